"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (needs oracle/_ref/libdfsref.so, i.e. /root/reference):

    python tests/golden/make_golden.py

Every array here is produced by the reference library's own public functions
through oracle/ref_harness.cpp. The oracle (oracle/dfs_oracle.c) and the CUDA
product are then checked against these files on machines without
/root/reference (the GPU box). Config shorthand follows SURVEY.md §8.
"""
from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle import fnv1a64_np, ref  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))

CONFIGS = {  # name: (dims, H, d, gamma)
    "T": ((4, 8, 8), 2, 64, 0.5),
    "C": ((13, 30, 45), 48, 64, 0.2),
    "W4": ((21, 30, 52), 40, 128, 0.15),
    "HY": ((33, 45, 80), 24, 128, 0.1),
    "W7": ((21, 45, 80), 40, 128, 0.3),
}


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round fp32 -> bf16 (RNE) -> fp32, the GPU input convention."""
    u = np.ascontiguousarray(x, np.float32).view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)


def head_inputs(dims, d, layer, head, smooth=4.0, seed=1):
    s = ref.derive_seed(seed, [layer, head])
    return [bf16_round(x) for x in ref.gen_video_field(dims, d, smooth, s)]


def perms():
    out = {}
    for name, (dims, _, _, _) in CONFIGS.items():
        fwd = ref.hilbert3d_order(dims)
        inv = ref.invert_permutation(fwd)
        out[f"{name}_head"] = fwd[:256].copy()
        out[f"{name}_tail"] = fwd[-256:].copy()
        out[f"{name}_fnv"] = np.array([fnv1a64_np(fwd), fnv1a64_np(inv)])
    # every ordering on a few small / ragged lattices
    for dims in [(1, 1, 1), (1, 1, 4), (2, 2, 2), (3, 5, 7), (5, 6, 7), (4, 8, 8), (1, 4, 8), (9, 3, 2)]:
        for o in ("raster", "hilbert2d", "block3d", "hilbert3d"):
            out[f"order_{o}_{dims[0]}x{dims[1]}x{dims[2]}"] = ref.order_tokens(o, dims)
    np.savez_compressed(os.path.join(OUT, "perms.npz"), **out)


def tiny():
    """Config T end to end for both heads: inputs, scores, mask, outputs."""
    dims, H, d, g = CONFIGS["T"]
    fwd = ref.hilbert3d_order(dims)
    out = {"fwd": fwd}
    for h in range(H):
        q, k, v = head_inputs(dims, d, 0, h)
        rq, rk, rv = (ref.apply_permutation(fwd, x) for x in (q, k, v))
        s = ref.block_scores(rq, rk, 64, 16)
        bits = ref.topk_select(s, g, 64)
        o = ref.block_sparse_attention(rq, rk, rv, bits, s.shape[0], 64)
        out[f"q{h}"], out[f"k{h}"], out[f"v{h}"] = q, k, v
        out[f"sub{h}"] = ref.subblock_scores(rq, rk, 64, 16)
        out[f"S{h}"], out[f"bits{h}"], out[f"o{h}"] = s, bits, o
        out[f"dense{h}"] = ref.full_attention_output(q, k, v)
    np.savez_compressed(os.path.join(OUT, "tiny.npz"), **out)


def cogvideo_head0():
    """Config C, layer 0 head 0: block scores, mask, and output rows of 3 query blocks."""
    dims, _, d, g = CONFIGS["C"]
    fwd = ref.hilbert3d_order(dims)
    q, k, v = head_inputs(dims, d, 0, 0)
    rq, rk, rv = (ref.apply_permutation(fwd, x) for x in (q, k, v))
    s = ref.block_scores(rq, rk, 128, 16)
    bits = ref.topk_select(s, g, 128)
    o = ref.block_sparse_attention(rq, rk, rv, bits, s.shape[0], 128)
    rows = np.r_[0:128, 64 * 128:65 * 128, (s.shape[0] - 1) * 128:rq.shape[0]]
    np.savez_compressed(os.path.join(OUT, "cogvideo_h0.npz"), S=s, bits=bits, rows=rows,
                        o_rows=o[rows], o_fnv=np.array([fnv1a64_np(o)]),
                        q_fnv=np.array([fnv1a64_np(q)]))


def kats():
    """Small known-answer cases restated from the reference unit tests."""
    out = {}
    rng = np.random.default_rng(1234)
    # ragged attention / score cases across odd geometry (test_attention.cpp:124-200 style)
    cases = []
    for i, (n, d, b, bs) in enumerate([(5, 3, 4, 2), (37, 8, 8, 4), (100, 16, 16, 4), (64, 64, 64, 16),
                                       (300, 64, 64, 16), (257, 128, 128, 16), (129, 64, 64, 64)]):
        q, k, v = (bf16_round(rng.standard_normal((n, d)).astype(np.float32)) for _ in range(3))
        s = ref.block_scores(q, k, b, bs)
        m = s.shape[0]
        g = [0.5, 0.3, 0.6, 1.0, 0.34, 0.5, 0.7][i]
        bits = ref.topk_select(s, g, b)
        out[f"c{i}_q"], out[f"c{i}_k"], out[f"c{i}_v"] = q, k, v
        out[f"c{i}_S"], out[f"c{i}_bits"] = s, bits
        out[f"c{i}_o"] = ref.block_sparse_attention(q, k, v, bits, m, b)
        out[f"c{i}_meta"] = np.array([n, d, b, bs, g])
        cases.append(i)
    out["cases"] = np.array(cases)
    # tie-heavy top-K rows (test_mask_builder.cpp:210-262)
    ties = rng.integers(0, 4, size=(50, 50)).astype(np.float64) / 4.0
    for g in (0.02, 0.1, 0.37, 0.5, 1.0):
        out[f"ties_{g}"] = ref.topk_select(ties, g, 16)
    out["ties"] = ties
    # cross attention (Nq != Nk) through full_attention_output
    q = bf16_round(rng.standard_normal((77, 64)).astype(np.float32))
    k = bf16_round(rng.standard_normal((200, 64)).astype(np.float32))
    v = bf16_round(rng.standard_normal((200, 64)).astype(np.float32))
    out["x_q"], out["x_k"], out["x_v"] = q, k, v
    out["x_o"] = ref.full_attention_output(q, k, v)
    np.savez_compressed(os.path.join(OUT, "kats.npz"), **out)


def schedules():
    out = {}
    cases = {
        "default": dict(total=50, warmup=0.25, budgets=(0.3, 0.2, 0.1), phase=0.25, interval=12),
        "w4": dict(total=50, warmup=0.25, budgets=(0.15,), phase=0.75, interval=12),
        "w7": dict(total=50, warmup=0.25, budgets=(0.3, 0.2, 0.1), phase=0.25, interval=6),
        "odd": dict(total=23, warmup=0.2, budgets=(0.5, 0.25), phase=0.4, interval=3),
        "one": dict(total=1, warmup=0.0, budgets=(0.1,), phase=1.0, interval=1),
    }
    for name, c in cases.items():
        b, u, ws, pl = ref.schedule(**c)
        out[f"{name}_budget"], out[f"{name}_update"] = b, u
        out[f"{name}_meta"] = np.array([ws, pl])
    np.savez_compressed(os.path.join(OUT, "schedules.npz"), **out)


def trajectory():
    """cmd_run-style trajectory (commands.cpp:221-319) at a small lattice: rows + masks."""
    import ctypes as C

    lib = ref.lib
    fn = lib.dfsref_run_trajectory
    fn.restype = C.c_int
    dims, d, L, H, T = (2, 8, 16), 16, 2, 2, 20
    b, bs = 32, 8
    budgets = np.array([0.5, 0.25], np.float64)
    n = dims[0] * dims[1] * dims[2]
    m = -(-n // b)
    mb = (m * m + 7) // 8
    rows = T * L * H
    rb, rsp = np.zeros(rows), np.zeros(rows)
    rf = np.zeros(rows, np.uint8)
    masks = np.zeros((rows, mb), np.uint8)
    out00 = np.zeros((T, n, d), np.float32)
    dense = np.array([1], np.int32)
    P = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    rc = fn(3, C.c_int64(dims[0]), C.c_int64(dims[1]), C.c_int64(dims[2]), C.c_int64(d), L, H, T,
            C.c_double(0.2), P(budgets), 2, C.c_double(0.4), 3, C.c_int64(b), C.c_int64(bs),
            C.c_uint64(1), C.c_double(4.0), C.c_double(2.0), C.c_double(0.0), 2, P(dense), 1,
            P(rb), P(rsp), P(rf), P(masks), P(out00))
    assert rc == 0, ref._err().decode()
    np.savez_compressed(os.path.join(OUT, "trajectory.npz"), budget=rb, sparsity=rsp, flags=rf,
                        masks=masks, out00=out00,
                        meta=np.array([dims[0], dims[1], dims[2], d, L, H, T, b, bs]),
                        budgets=budgets, dense_layers=dense)


if __name__ == "__main__":
    assert ref is not None, "needs oracle/_ref/libdfsref.so (make -C oracle ref)"
    for fn in (perms, tiny, cogvideo_head0, kats, schedules, trajectory):
        fn()
        print("wrote", fn.__name__)
