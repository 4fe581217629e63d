"""Host-side mirror of the reference's dfs:: operator API over CUDA tensors.

Every function here is a thin host wrapper: argument checks that raise the
reference's exception types (ValueError = std::invalid_argument, IndexError =
std::out_of_range), device buffer plumbing with torch, and one or more calls
through the C ABI (include/dfs_gpu.h) into the sm_100a kernels. Nothing
computes on the CPU. Names and argument meaning follow
/root/reference/proj/include/dfs/{curve,mask_builder,attention,scheduler}.hpp.

Tensors: token matrices are CUDA tensors [N, d] (one head, the reference's
Matrix) or [N, H, d] / [H, N, d] (batched heads); fp32 or bf16. Permutations are
int32 CUDA tensors holding the u32 forward map. Block masks are BlockMask
objects wrapping the reference's bit payload (MSB-first, row-major) on device.
"""
from __future__ import annotations

import ctypes as C
import math
import threading
from dataclasses import dataclass, field

import torch

from . import _capi as capi

# --------------------------------------------------------------------------- #
# handle / stream plumbing                                                     #
# --------------------------------------------------------------------------- #


class Handle:
    """Owns a dfs_handle (workspaces, permutation cache, device mask cache)."""

    def __init__(self, device: int | None = None):
        if not torch.cuda.is_available():
            raise RuntimeError("DFSAttn-B200 needs a CUDA device (no CPU fallback)")
        self.device = torch.cuda.current_device() if device is None else int(device)
        ptr = C.c_void_p()
        capi.call("dfs_handle_create", C.byref(ptr), self.device)
        self.ptr = ptr

    def close(self):
        if getattr(self, "ptr", None):
            capi.lib.dfs_handle_destroy(self.ptr)
            self.ptr = None

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            self.close()
        except Exception:
            pass

    def set_option(self, option: int, value: int) -> None:
        capi.call("dfs_handle_set_option", self.ptr, int(option), int(value))

    def workspace_bytes(self) -> int:
        n = C.c_int64()
        capi.call("dfs_handle_workspace_bytes", self.ptr, C.byref(n))
        return n.value


_tls = threading.local()


def default_handle() -> Handle:
    """One handle per thread (the C ABI's threading contract, scheduler.hpp:52-53)."""
    h = getattr(_tls, "handle", None)
    if h is None:
        h = Handle()
        _tls.handle = h
    return h


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def _ptr(t: torch.Tensor | None):
    return C.c_void_p(0 if t is None else t.data_ptr())


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return capi.DFS_BF16
    if t.dtype == torch.float32:
        return capi.DFS_F32
    raise ValueError(f"unsupported dtype {t.dtype}; use float32 or bfloat16")


def _check_cuda(*ts):
    for t in ts:
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError("expected CUDA tensors (the DFSAttn-B200 path has no CPU fallback)")


# --------------------------------------------------------------------------- #
# value types (block_mask.hpp, curve.hpp, grid.hpp)                            #
# --------------------------------------------------------------------------- #


@dataclass(frozen=True)
class GridDims:
    frames: int = 1
    height: int = 1
    width: int = 1

    def token_count(self) -> int:
        return self.frames * self.height * self.width

    def validate(self):  # grid.hpp:21-28
        if self.frames < 1 or self.height < 1 or self.width < 1:
            raise ValueError("GridDims: extents must be >= 1")
        if self.frames > (1 << 31) // self.height // self.width:
            raise ValueError("GridDims: token count overflows index range")


@dataclass
class Permutation:
    forward: torch.Tensor  # int32 CUDA [N]: raster index at reordered position i
    label: str = "raster"

    def size(self) -> int:
        return int(self.forward.numel())


@dataclass
class ScoringParams:  # mask_builder.hpp:11-23
    block_size: int = 128
    sub_block_size: int = 16

    def subs_per_block(self) -> int:
        return self.block_size // self.sub_block_size

    def validate(self):
        if self.sub_block_size < 1 or self.block_size < self.sub_block_size:
            raise ValueError("ScoringParams: need 1 <= sub_block_size <= block_size")
        if self.block_size % self.sub_block_size:
            raise ValueError("ScoringParams: sub_block_size must divide block_size")


def block_count_for(tokens: int, block_size: int) -> int:  # block_mask.hpp:10-13
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    return (tokens + block_size - 1) // block_size


@dataclass
class BlockMask:
    """M x M block mask; `bits` is the reference payload (uint8 CUDA tensor)."""

    bits: torch.Tensor
    block_count: int
    block_size: int

    @staticmethod
    def byte_size(m: int) -> int:
        return (m * m + 7) // 8

    @classmethod
    def full(cls, m: int, b: int, selected: bool, device=None) -> "BlockMask":
        if m < 1 or b < 1:
            raise ValueError("BlockMask: block_count and block_size must be >= 1")
        dense = torch.full((m, m), bool(selected), dtype=torch.bool)
        return cls.from_dense(dense, b, device)

    @classmethod
    def from_dense(cls, dense: torch.Tensor, b: int, device=None) -> "BlockMask":
        m = dense.shape[0]
        flat = torch.zeros(((m * m + 7) // 8) * 8, dtype=torch.uint8)
        flat[: m * m] = dense.reshape(-1).to(torch.uint8).cpu()
        weights = torch.tensor([128, 64, 32, 16, 8, 4, 2, 1], dtype=torch.int32)
        packed = (flat.view(-1, 8).to(torch.int32) * weights).sum(1).to(torch.uint8)
        dev = device if device is not None else torch.device("cuda", torch.cuda.current_device())
        return cls(packed.to(dev), m, b)

    def to_dense(self) -> torch.Tensor:
        m = self.block_count
        b = self.bits.to(torch.int32).cpu()
        bits = torch.stack([(b >> (7 - j)) & 1 for j in range(8)], 1).reshape(-1)[: m * m]
        return bits.reshape(m, m).bool()

    def get(self, u: int, v: int) -> bool:
        idx = u * self.block_count + v
        return bool((int(self.bits[idx >> 3]) >> (7 - (idx & 7))) & 1)

    def selected_count(self) -> int:
        return int(self.to_dense().sum())

    def row_empty(self, u: int) -> bool:
        return not bool(self.to_dense()[u].any())

    def __eq__(self, other):
        return (isinstance(other, BlockMask) and self.block_count == other.block_count
                and self.block_size == other.block_size and torch.equal(self.bits.cpu(), other.bits.cpu()))


def realized_sparsity(mask: BlockMask) -> float:  # metrics.cpp:39-42
    m = mask.block_count
    return 1.0 - mask.selected_count() / float(m * m)


# --------------------------------------------------------------------------- #
# reorder (curve.hpp)                                                          #
# --------------------------------------------------------------------------- #


def _dims(d) -> GridDims:
    return d if isinstance(d, GridDims) else GridDims(*[int(x) for x in d])


def order_tokens(ordering: str, dims) -> Permutation:
    """curve.hpp:48 order_tokens — K1 on device."""
    dims = _dims(dims)
    dims.validate()
    if ordering not in capi.ORDERINGS:
        raise ValueError(f"unknown ordering: {ordering}")
    fwd = torch.empty(dims.token_count(), dtype=torch.int32, device="cuda")
    capi.call("dfs_order_tokens", capi.ORDERINGS[ordering], dims.frames, dims.height, dims.width,
              _ptr(fwd), None, _stream())
    return Permutation(fwd, ordering)


def raster_order(dims) -> Permutation:
    return order_tokens("raster", dims)


def hilbert3d_order(dims) -> Permutation:
    return order_tokens("hilbert3d", dims)


def hilbert2d_order(dims) -> Permutation:
    return order_tokens("hilbert2d", dims)


def block3d_order(dims) -> Permutation:
    return order_tokens("block3d", dims)


def invert_permutation(perm: Permutation) -> Permutation:
    """curve.hpp:53 — inverse.forward[perm.forward[i]] == i."""
    inv = torch.empty_like(perm.forward)
    capi.call("dfs_invert_permutation", _ptr(perm.forward), perm.size(), _ptr(inv), _stream())
    return Permutation(inv, perm.label)


def validate_permutation(forward: torch.Tensor) -> None:
    """curve.hpp:27 — raises ValueError unless forward is a bijection on [0, N)."""
    if forward.numel() == 0:
        raise ValueError("permutation: empty")
    ok = C.c_int()
    capi.call("dfs_validate_permutation", default_handle().ptr, _ptr(forward), forward.numel(), C.byref(ok),
              _stream())
    if not ok.value:
        raise ValueError("permutation: not a bijection")


def _as_heads(x: torch.Tensor):
    """[N, d] -> (N, 1, d); [N, H, d] stays NHD."""
    if x.dim() == 2:
        return x.shape[0], 1, x.shape[1]
    if x.dim() == 3:
        return x.shape[0], x.shape[1], x.shape[2]
    raise ValueError("expected a [N, d] or [N, H, d] tensor")


def apply_permutation(perm: Permutation, x: torch.Tensor) -> torch.Tensor:
    """curve.hpp:50 — row i of the result is row forward[i] of x (K2 gather)."""
    _check_cuda(x)
    n, h, d = _as_heads(x)
    if perm.size() != n:
        raise ValueError("apply_permutation: length mismatch")
    x = x.contiguous()
    out = torch.empty_like(x)
    capi.call("dfs_permute_rows", _ptr(x), capi.DFS_NHD, _ptr(out), capi.DFS_NHD, _dtype_code(x),
              _ptr(perm.forward), n, h, d, None, 1, None, _stream())
    return out


def unpermute(perm: Permutation, x: torch.Tensor) -> torch.Tensor:
    """apply_permutation(invert_permutation(perm), x) without materialising the inverse (K6)."""
    _check_cuda(x)
    n, h, d = _as_heads(x)
    if perm.size() != n:
        raise ValueError("apply_permutation: length mismatch")
    x = x.contiguous()
    out = torch.empty_like(x)
    capi.call("dfs_unpermute_rows", _ptr(x), capi.DFS_NHD, _ptr(out), capi.DFS_NHD, _dtype_code(x),
              _ptr(perm.forward), n, h, d, _stream())
    return out


# --------------------------------------------------------------------------- #
# score / mask (mask_builder.hpp)                                              #
# --------------------------------------------------------------------------- #


def _identity(n: int, device) -> torch.Tensor:
    return torch.arange(n, dtype=torch.int32, device=device)


def _pool_heads(x: torch.Tensor, pool: int, layout: int) -> torch.Tensor:
    """fp32 [H, ceil(N/pool), d] sub-block means (K2's pooled output, identity order)."""
    if layout == capi.DFS_HND:
        h, n, d = x.shape
    else:
        n, h, d = _as_heads(x)
    x = x.contiguous()
    scratch = torch.empty_like(x)
    pooled = torch.empty((h, (n + pool - 1) // pool, d), dtype=torch.float32, device=x.device)
    flag = torch.zeros(1, dtype=torch.int32, device=x.device)
    capi.call("dfs_permute_rows", _ptr(x), layout, _ptr(scratch), layout, _dtype_code(x),
              _ptr(_identity(n, x.device)), n, h, d, _ptr(pooled), pool, _ptr(flag), _stream())
    if int(flag.item()):
        raise ValueError("attention: non-finite input")
    return pooled


def mean_pool(x: torch.Tensor, pool: int) -> torch.Tensor:
    """mask_builder.hpp:27 — [N, d] -> [ceil(N/pool), d] fp32, zero-padded, divided by pool."""
    _check_cuda(x)
    if pool < 1:
        raise ValueError("mean_pool: pool must be >= 1")
    if x.shape[0] < 1:
        raise ValueError("mean_pool: empty input")
    p = _pool_heads(x, pool, capi.DFS_NHD)
    return p[0] if x.dim() == 2 else p.transpose(0, 1).contiguous()


def block_scores(q: torch.Tensor, k: torch.Tensor, params: ScoringParams, layout: int = capi.DFS_NHD
                 ) -> torch.Tensor:
    """mask_builder.hpp:54 — fp64 [M, M] (or [H, M, M] for batched heads)."""
    params.validate()
    _check_cuda(q, k)
    if q.shape != k.shape:
        raise ValueError("subblock_scores: head dims differ" if q.shape[-1] != k.shape[-1]
                         else "build_mask: q and k row counts differ")
    if layout == capi.DFS_HND:
        h, n, d = q.shape
    else:
        n, h, d = _as_heads(q)
    pq = _pool_heads(q, params.sub_block_size, layout)
    pk = _pool_heads(k, params.sub_block_size, layout)
    m = block_count_for(n, params.block_size)
    s = torch.empty((h, m, m), dtype=torch.float64, device=q.device)
    capi.call("dfs_score_blocks", default_handle().ptr, _ptr(pq), _ptr(pk), h, n, d, params.block_size,
              params.sub_block_size, _ptr(s), _stream())
    return s[0] if (q.dim() == 2) else s


def topk_count(budget: float, block_count: int) -> int:
    """mask_builder.hpp:38 — K = min(M, max(1, llround(budget*M)))."""
    k = C.c_int64()
    capi.call("dfs_topk_count", float(budget), int(block_count), C.byref(k))
    return k.value


def topk_lut(scores: torch.Tensor, budget: float) -> torch.Tensor:
    """Per (head, row) ascending K best key blocks as int32 [.., M, K] (K4)."""
    s3 = scores if scores.dim() == 3 else scores.unsqueeze(0)
    if s3.shape[-1] != s3.shape[-2] or s3.shape[-1] < 1:
        raise ValueError("topk_select: scores must be square and non-empty")
    h, m, _ = s3.shape
    k = topk_count(budget, m)
    s3 = s3.to(torch.float64).contiguous()
    lut = torch.empty((h, m, k), dtype=torch.int32, device=s3.device)
    capi.call("dfs_topk_select", _ptr(s3), h, m, k, _ptr(lut), None, _stream())
    return lut if scores.dim() == 3 else lut[0]


def topk_select(scores: torch.Tensor, budget: float, block_size: int):
    """mask_builder.hpp:51 — BlockMask (list of BlockMask for [H, M, M] scores)."""
    s3 = scores if scores.dim() == 3 else scores.unsqueeze(0)
    if s3.shape[-1] != s3.shape[-2] or s3.shape[-1] < 1:
        raise ValueError("topk_select: scores must be square and non-empty")
    h, m, _ = s3.shape
    k = topk_count(budget, m)
    s3 = s3.to(torch.float64).contiguous()
    nb = BlockMask.byte_size(m)
    bits = torch.empty((h, nb), dtype=torch.uint8, device=s3.device)
    capi.call("dfs_topk_select", _ptr(s3), h, m, k, None, _ptr(bits), _stream())
    masks = [BlockMask(bits[i].clone(), m, block_size) for i in range(h)]
    return masks if scores.dim() == 3 else masks[0]


def build_mask(q: torch.Tensor, k: torch.Tensor, params: ScoringParams, budget: float):
    """mask_builder.hpp:57 — the full scoring/selection chain."""
    if q.shape[0] != k.shape[0]:
        raise ValueError("build_mask: q and k row counts differ")
    return topk_select(block_scores(q, k, params), budget, params.block_size)


# --------------------------------------------------------------------------- #
# attention (attention.hpp)                                                    #
# --------------------------------------------------------------------------- #


def _attn_call(q, k, v, out, heads, nq, nk, d, block, blk_ptr, blk_idx, in_layout, out_layout,
               out_rows=None, force_generic=False, scale=0.0, in_rows=None):
    a = capi.AttnArgs(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), _dtype_code(q), in_layout,
                      out_layout, heads, nq, nk, d, block,
                      0 if blk_ptr is None else blk_ptr.data_ptr(),
                      0 if blk_idx is None else blk_idx.data_ptr(),
                      0 if out_rows is None else out_rows.data_ptr(), float(scale), int(force_generic),
                      0 if v.shape[-1] == d else v.shape[-1], 0 if in_rows is None else in_rows.data_ptr())
    capi.call("dfs_sparse_attn_fwd", default_handle().ptr, C.byref(a), _stream())


def _check_qkv(q, k, v):  # attention.cpp:14-21
    _check_cuda(q, k, v)
    if q.dim() != k.dim() or k.dim() != v.dim() or q.dim() not in (2, 3):
        raise ValueError("attention: expected [N, d] or [N, H, d] tensors")
    if q.shape[-1] != k.shape[-1]:
        raise ValueError("attention: q and k head dims differ")
    if k.shape[0] != v.shape[0]:
        raise ValueError("attention: k and v row counts differ")
    if q.dim() == 3 and not (q.shape[1] == k.shape[1] == v.shape[1]):
        raise ValueError("attention: q, k, v head counts differ")
    if v.shape[-1] != q.shape[-1] and q.dtype != torch.float32:
        raise ValueError("attention: dv != d only on the fp32 path")
    if q.shape[0] < 1 or k.shape[0] < 1 or q.shape[-1] < 1:
        raise ValueError("attention: empty input")
    if q.dtype != k.dtype or k.dtype != v.dtype:
        raise ValueError("attention: q, k, v dtypes differ")
    for t in (q, k, v):
        if not bool(torch.isfinite(t).all()):
            raise ValueError("attention: non-finite input")


def mask_to_csr(masks, m: int):
    """BlockMask(s) -> device CSR (blk_ptr [H*M+1], blk_idx); ValueError on an empty row."""
    ms = masks if isinstance(masks, (list, tuple)) else [masks]
    h = len(ms)
    bits = torch.stack([mm.bits for mm in ms]).contiguous()
    ptr = torch.empty(h * m + 1, dtype=torch.int32, device=bits.device)
    idx = torch.empty(max(h * m * m, 1), dtype=torch.int32, device=bits.device)
    nnz = C.c_int64()
    capi.call("dfs_mask_bits_to_csr", default_handle().ptr, _ptr(bits), h, m, _ptr(ptr), _ptr(idx),
              C.byref(nnz), _stream())
    return ptr, idx[: max(nnz.value, 1)]


def block_sparse_attention(q, k, v, mask, force_generic: bool = False) -> torch.Tensor:
    """attention.hpp:32 — softmax over the selected key blocks only (K5).

    q, k, v: [N, d] with a BlockMask, or [N, H, d] with a list of H BlockMasks.
    """
    _check_qkv(q, k, v)
    if q.shape[0] != k.shape[0]:
        raise ValueError("block_sparse_attention: q and k row counts differ")
    n, h, d = _as_heads(q)
    ms = mask if isinstance(mask, (list, tuple)) else [mask]
    if len(ms) != h:
        raise ValueError("block_sparse_attention: need one mask per head")
    b, m = ms[0].block_size, ms[0].block_count
    for mm in ms:
        if block_count_for(n, mm.block_size) != mm.block_count or mm.block_size != b:
            raise ValueError("block mask geometry inconsistent with sequence length")
    ptr, idx = mask_to_csr(ms, m)
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    out = q.new_empty(q.shape[:-1] + (v.shape[-1],))
    _attn_call(q, k, v, out, h, n, n, d, b, ptr, idx, capi.DFS_NHD, capi.DFS_NHD, force_generic=force_generic)
    return out


def full_attention_output(q, k, v, block: int = 128, force_generic: bool = False) -> torch.Tensor:
    """attention.hpp:23 — dense softmax attention, Nq != Nk allowed (cross attention).

    Runs through the same K5 kernel with a full mask (blk_ptr = NULL)."""
    _check_qkv(q, k, v)
    nq, h, d = _as_heads(q)
    nk = k.shape[0]
    q, k, v = q.contiguous(), k.contiguous(), v.contiguous()
    out = q.new_empty(q.shape[:-1] + (v.shape[-1],))
    _attn_call(q, k, v, out, h, nq, nk, d, block, None, None, capi.DFS_NHD, capi.DFS_NHD,
               force_generic=force_generic)
    return out


def sparse_attention_csr(q, k, v, blk_ptr, blk_idx, block, layout=capi.DFS_HND, out_layout=None,
                         out_rows=None, out=None, force_generic=False, in_rows=None):
    """Batched K5 over all heads: q/k/v [H, N, d] (HND) or [N, H, d] (NHD) bf16.

    in_rows (NHD only): logical row i is raster row in_rows[i] (the reorder fused into K5)."""
    if in_rows is not None:  # q is the raster [N, H, d] tensor, gathered inside K5
        nq, h, d = q.shape
        nk = k.shape[1] if layout == capi.DFS_HND else k.shape[0]
    elif layout == capi.DFS_HND:
        h, nq, d = q.shape
        nk = k.shape[1]
    else:
        nq, h, d = q.shape
        nk = k.shape[0]
    out_layout = layout if out_layout is None else out_layout
    if out is None:
        out = torch.empty((h, nq, d) if out_layout == capi.DFS_HND else (nq, h, d), dtype=q.dtype,
                          device=q.device)
    _attn_call(q, k, v, out, h, nq, nk, d, block, blk_ptr, blk_idx, layout, out_layout, out_rows,
               force_generic, in_rows=in_rows)
    return out


def pool_gathered(x: torch.Tensor, perm: Permutation, pool: int, nonfinite: torch.Tensor | None = None):
    """K2 read-only: sub-block means of x [N, H, d] taken in `perm` order -> fp32 [H, ceil(N/pool), d]."""
    n, h, d = x.shape
    pooled = torch.empty((h, (n + pool - 1) // pool, d), dtype=torch.float32, device=x.device)
    capi.call("dfs_permute_rows", _ptr(x), capi.DFS_NHD, None, capi.DFS_HND, _dtype_code(x), _ptr(perm.forward),
              n, h, d, _ptr(pooled), pool, _ptr(nonfinite), _stream())
    return pooled


# --------------------------------------------------------------------------- #
# schedule + mask cache + Alg. 1 step (scheduler.hpp)                          #
# --------------------------------------------------------------------------- #


@dataclass
class ScheduleConfig:  # scheduler.hpp:22-28
    total_steps: int = 50
    warmup_fraction: float = 0.25
    phase_budgets: tuple = (0.3, 0.2, 0.1)
    phase_fraction: float = 0.25
    update_interval: int = 12


class SparsitySchedule:
    """scheduler.hpp:20-50 — evaluated by the library's host code (dfs_schedule_*)."""

    def __init__(self, config: ScheduleConfig | None = None, **kw):
        self.config = config or ScheduleConfig(**kw)
        c = self.config
        self._budgets = (C.c_double * max(len(c.phase_budgets), 1))(*c.phase_budgets)
        self._s = capi.Schedule(int(c.total_steps), float(c.warmup_fraction), self._budgets,
                                len(c.phase_budgets), float(c.phase_fraction), int(c.update_interval))
        w, p = C.c_int(), C.c_int()
        capi.call("dfs_schedule_info", C.byref(self._s), C.byref(w), C.byref(p))
        self._warmup, self._phase = w.value, p.value

    def budget_at(self, step: int):
        b = C.c_double()
        capi.call("dfs_schedule_budget_at", C.byref(self._s), int(step), C.byref(b))
        return None if b.value < 0 else b.value

    def is_update_step(self, step: int) -> bool:
        r = C.c_int()
        capi.call("dfs_schedule_is_update_step", C.byref(self._s), int(step), C.byref(r))
        return bool(r.value)

    def total_steps(self):
        return self.config.total_steps

    def warmup_steps(self):
        return self._warmup

    def first_sparse_step(self):
        return self._warmup

    def phase_length(self):
        return self._phase

    def update_interval(self):
        return self.config.update_interval


class MaskCache:
    """scheduler.hpp:54-71 — device-resident, keyed by (layer, head), owned by a Handle.

    Internally locked like the reference's (scheduler.cpp:58-83): a dfs_handle must not be
    used by two threads at once (dfs_gpu.h), so every call on the cache's handle —
    including run_step with this cache — holds `self.lock`."""

    def __init__(self, handle: Handle | None = None):
        self.handle = handle or Handle()
        self.lock = threading.RLock()

    def contains(self, layer: int, head: int) -> bool:
        f = C.c_int()
        with self.lock:
            capi.call("dfs_mask_cache_contains", self.handle.ptr, layer, head, C.byref(f))
        return bool(f.value)

    def find(self, layer: int, head: int):
        """-> (BlockMask, last_update_step) or None (a copy, like the reference)."""
        with self.lock:
            if not self.contains(layer, head):
                return None
            m, b, step = C.c_int64(), C.c_int64(), C.c_int()
            capi.call("dfs_mask_cache_info", self.handle.ptr, layer, head, C.byref(m), C.byref(b), C.byref(step))
            bits = torch.empty(BlockMask.byte_size(m.value), dtype=torch.uint8, device="cuda")
            capi.call("dfs_mask_cache_get", self.handle.ptr, layer, head, _ptr(bits), None, None, _stream())
            return BlockMask(bits, m.value, b.value), step.value

    def store(self, layer: int, head: int, mask: BlockMask, step: int):
        with self.lock:
            capi.call("dfs_mask_cache_store", self.handle.ptr, layer, head, _ptr(mask.bits), mask.block_count,
                      mask.block_size, step, _stream())

    def size(self) -> int:
        n = C.c_int64()
        with self.lock:
            capi.call("dfs_mask_cache_size", self.handle.ptr, C.byref(n))
        return n.value

    def empty(self) -> bool:
        return self.size() == 0

    def clear(self):
        with self.lock:
            capi.call("dfs_mask_cache_clear", self.handle.ptr)


def should_update(cache: MaskCache, layer: int, head: int, step: int, schedule: SparsitySchedule) -> bool:
    """scheduler.cpp:85-89."""
    if not cache.contains(layer, head):
        return True
    return schedule.is_update_step(step)


@dataclass
class StepStats:  # scheduler.hpp:78-85 (per head)
    dense: bool = True
    budget: float = 1.0
    mask_updated: list = field(default_factory=list)
    sparsity: list = field(default_factory=list)
    recall: list | None = None  # per head, when run_step(..., record_recall=True)


@dataclass
class QkPrologue:
    """QK-norm + RoPE fused into K2 (dfs_qk_prologue): q and k rows are RMS-normalised over d
    (x * weight / sqrt(mean(x^2) + eps)) and rotated by RoPE before they are reordered, pooled
    and attended. Weights: fp32 CUDA [d] (None: no norm); rope_cos / rope_sin: fp32 CUDA
    [N, d/2] by raster token; rope: "none" | "interleaved" (pairs 2i, 2i+1) | "half" (i, i+d/2)."""

    q_norm_weight: torch.Tensor | None = None
    k_norm_weight: torch.Tensor | None = None
    eps: float = 1e-6
    rope: str = "none"
    rope_cos: torch.Tensor | None = None
    rope_sin: torch.Tensor | None = None

    def c_args(self):
        for t in (self.q_norm_weight, self.k_norm_weight, self.rope_cos, self.rope_sin):
            if t is not None and (not t.is_cuda or t.dtype != torch.float32 or not t.is_contiguous()):
                raise ValueError("QkPrologue: weights and RoPE tables must be contiguous fp32 CUDA tensors")
        if self.rope not in capi.ROPE_LAYOUTS:
            raise ValueError(f"QkPrologue: unknown RoPE layout {self.rope}")
        return capi.QkPrologueArgs(_ptr(self.q_norm_weight).value, _ptr(self.k_norm_weight).value, float(self.eps),
                                   capi.ROPE_LAYOUTS[self.rope], _ptr(self.rope_cos).value,
                                   _ptr(self.rope_sin).value)

    def apply(self, x: torch.Tensor, which: str = "q") -> torch.Tensor:
        """The prologue alone on bf16 [N, H, d] raster rows (q or k weights) -> bf16 [N, H, d]."""
        n, h, d = x.shape
        out = torch.empty_like(x)
        a = self.c_args()
        capi.call("dfs_qk_prologue_apply", C.byref(a), 0 if which == "q" else 1, _ptr(x), _ptr(out), capi.DFS_NHD,
                  None, n, h, d, _stream())
        return out


def run_step(q, k, v, dims, params: ScoringParams, schedule: SparsitySchedule, cache: MaskCache, layer: int,
             step: int, force_dense: bool = False, perm: Permutation | None = None, out=None,
             record_recall: bool = False, prologue: QkPrologue | None = None):
    """scheduler.hpp:93 run_step for ALL heads of one layer: q, k, v [N, H, d] raster order.

    bf16 is the performance path; fp32 runs the compatibility kernels up to 4096 tokens
    (the reference's fp64 arithmetic) and the tcgen05 kernels past it. Non-finite input
    raises ValueError before anything is scored, cached or written (attention.cpp:19-20).
    Returns (out [N, H, d], StepStats)."""
    _check_cuda(q, k, v)
    if q.dtype not in (torch.bfloat16, torch.float32) or k.dtype != q.dtype or v.dtype != q.dtype:
        raise ValueError("run_step: q, k, v must all be bf16 (performance path) or all fp32")
    if q.dim() != 3 or k.shape != q.shape or v.shape[:2] != q.shape[:2]:
        raise ValueError("run_step: expected q, k [N, H, d] and v [N, H, dv] with the same N and H")
    if not (q.is_contiguous() and k.is_contiguous() and v.is_contiguous()):
        raise ValueError("run_step: q, k, v must be contiguous [N, H, d] tensors")
    n, h, d = q.shape
    dv = v.shape[2]
    dims = _dims(dims)
    if perm is None and dims.token_count() != n:
        raise ValueError("run_step: permutation length does not match token count")
    if perm is not None and perm.size() != n:
        raise ValueError("run_step: permutation length does not match token count")
    out = torch.empty((n, h, dv), dtype=q.dtype, device=q.device) if out is None else out
    if out.shape != (n, h, dv) or out.dtype != q.dtype or not out.is_contiguous():
        raise ValueError("run_step: out must be a contiguous [N, H, dv] tensor of the input dtype")
    dense, budget = C.c_int(), C.c_double()
    upd = (C.c_int * h)()
    spars = (C.c_double * h)()
    rec = (C.c_double * h)() if record_recall else None
    a = capi.StepArgs(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), n, h, d,
                      0 if perm is None else perm.forward.data_ptr(), dims.frames, dims.height, dims.width,
                      params.block_size, params.sub_block_size, layer, step, int(force_dense),
                      None, C.pointer(dense), C.pointer(budget),
                      C.cast(upd, C.POINTER(C.c_int)), C.cast(spars, C.POINTER(C.c_double)),
                      C.cast(rec, C.POINTER(C.c_double)) if rec is not None else None, _dtype_code(q), dv, None)
    pro = prologue.c_args() if prologue is not None else None
    if pro is not None:
        a.prologue = C.cast(C.pointer(pro), C.c_void_p)
    with cache.lock:
        capi.call("dfs_run_step", cache.handle.ptr, C.byref(schedule._s), C.byref(a), _stream())
    stats = StepStats(bool(dense.value), budget.value, [bool(x) for x in upd], list(spars),
                      list(rec) if rec is not None else None)
    return out, stats


def block_recall(q, k, blk_ptr, blk_idx, layout=capi.DFS_HND, q_rows=None):
    """attention_recall(attention_scores(q, k), mask) per head at any N (streamed, no N x N).

    q, k: bf16 [H, N, d] (HND) or [N, H, d] (NHD); q_rows: q is raster NHD gathered by row."""
    if q_rows is not None or layout == capi.DFS_NHD:
        n, h, d = q.shape
    else:
        h, n, d = q.shape
    rec = (C.c_double * h)()
    capi.call("dfs_block_recall", default_handle().ptr, _ptr(q), _ptr(k), layout, _ptr(q_rows), h, n, d,
              _ptr(blk_ptr), _ptr(blk_idx), C.cast(rec, C.POINTER(C.c_double)), _stream())
    return list(rec)


# --------------------------------------------------------------------------- #
# decomposed batched pipeline (used by bench.py to time each kernel)           #
# --------------------------------------------------------------------------- #


def permute_to_hnd(x: torch.Tensor, perm: Permutation, pool: int = 0, nonfinite: torch.Tensor | None = None):
    """K2: [N, H, d] raster -> [H, N, d] reordered (+ fp32 pooled [H, ceil(N/pool), d] when pool > 0)."""
    n, h, d = x.shape
    out = torch.empty((h, n, d), dtype=x.dtype, device=x.device)
    pooled = None
    if pool > 0:
        pooled = torch.empty((h, (n + pool - 1) // pool, d), dtype=torch.float32, device=x.device)
    capi.call("dfs_permute_rows", _ptr(x), capi.DFS_NHD, _ptr(out), capi.DFS_HND, _dtype_code(x), _ptr(perm.forward),
              n, h, d, _ptr(pooled), max(pool, 1), _ptr(nonfinite), _stream())
    return out, pooled


def score_pooled(pq: torch.Tensor, pk: torch.Tensor, n: int, params: ScoringParams, out: torch.Tensor | None = None):
    """K3 on pooled inputs [H, ceil(N/Bs), d] -> fp64 [H, M, M]."""
    h, _, d = pq.shape
    m = block_count_for(n, params.block_size)
    s = torch.empty((h, m, m), dtype=torch.float64, device=pq.device) if out is None else out
    capi.call("dfs_score_blocks", default_handle().ptr, _ptr(pq), _ptr(pk), h, n, d, params.block_size,
              params.sub_block_size, _ptr(s), _stream())
    return s


def lut_row_ptr(heads: int, m: int, k: int, device="cuda") -> torch.Tensor:
    ptr = torch.empty(heads * m + 1, dtype=torch.int32, device=device)
    capi.call("dfs_lut_row_ptr", heads, m, k, _ptr(ptr), _stream())
    return ptr
