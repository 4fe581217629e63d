"""Parity pins at the headline shapes: the product path (dfs.run_step through the
C ABI, tcgen05 K3/K5) against the C oracle on inputs from the reference's own
generator (oracle ``gen_video_field``, bf16-rounded: SURVEY.md §8(d)).

Shared by tests/test_gpu_parity_pins.py (the assertions) and
tools/parity_report.py (the same numbers written to profiles/). Test
infrastructure: imports the oracle, never shipped.

Per head it reports
  * score_err     max|S_gpu - S_ref| / max|S_ref| of the device K3 block scores
                  (mask_builder.cpp:30-80) vs the oracle's fp64 block_scores;
  * bit_agree     fraction of the M^2 mask bits equal (device mask vs oracle mask);
  * set_overlap   |I_gpu ∩ I_ref| / |I_ref| over all rows (selected-set overlap);
  * rows_equal    fraction of query-block rows whose selected sets are identical;
  * k4_exact      the device mask is the oracle's top-K of the DEVICE scores
                  (selection bit-exact given identical scores, mask_builder.cpp:91-113);
  * out_err       max|O - O_ref| / max|O_ref| over sampled query blocks (first,
                  middle, partial last), O_ref = the oracle's block_sparse_attention
                  (attention.cpp:125-159) under the ORACLE's mask, fp64 arithmetic;
  * out_err_own   the same under the device's own mask (isolates K5 from K3).
"""
from __future__ import annotations

import numpy as np

from oracle import mask_bits_to_dense, ora

from tests.golden.make_golden import bf16_round

# name: (dims, d, gamma, smoothness, heads)
CASES = {
    "W7_g0.30": ((21, 45, 80), 128, 0.30, 4.0, 3),
    "W7_g0.05": ((21, 45, 80), 128, 0.05, 4.0, 3),
    "HY_iid": ((33, 45, 80), 128, 0.10, 0.0, 2),
    "HY_smooth": ((33, 45, 80), 128, 0.10, 4.0, 2),
    "C_iid": ((13, 30, 45), 64, 0.20, 0.0, 2),
}


def head_inputs(dims, d, smooth, heads, seed=1, layer=0):
    out = []
    for h in range(heads):
        q, k, v = (bf16_round(x) for x in ora.gen_video_field(dims, d, smooth, ora.derive_seed(seed, [layer, h])))
        out.append((q, k, v))
    return out


def run_case(name, torch, dfs, block=128, sub=16):
    dims, d, gamma, smooth, heads = CASES[name]
    n = int(np.prod(dims))
    m = -(-n // block)
    hin = head_inputs(dims, d, smooth, heads)
    Q, K, V = (torch.from_numpy(np.stack([x[i] for x in hin], 1)).to(torch.bfloat16).cuda() for i in range(3))
    params = dfs.ScoringParams(block, sub)
    sched = dfs.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(gamma,), phase_fraction=1.0,
                                 update_interval=1)
    cache = dfs.MaskCache()
    out, stats = dfs.run_step(Q, K, V, dims, params, sched, cache, layer=0, step=0)
    perm = dfs.hilbert3d_order(dims)
    S_dev = dfs.block_scores(dfs.apply_permutation(perm, Q), dfs.apply_permutation(perm, K), params).cpu().numpy()
    if S_dev.ndim == 2:
        S_dev = S_dev[None]
    out = out.float().cpu().numpy()
    fwd = ora.hilbert3d_order(dims)
    assert (perm.forward.cpu().numpy().astype(np.uint32) == fwd).all()
    sample_blocks = sorted({0, m // 2, m - 1})
    res = {"case": name, "dims": list(dims), "n": n, "d": d, "gamma": gamma, "smoothness": smooth,
           "M": m, "K": ora.topk_count(gamma, m), "heads": []}
    for h in range(heads):
        q, k, v = hin[h]
        rq, rk, rv = (ora.apply_permutation(fwd, x) for x in (q, k, v))
        S_ref = ora.block_scores(rq, rk, block, sub)
        bits_ref = ora.topk_select(S_ref, gamma)
        dense_ref = mask_bits_to_dense(bits_ref, m)
        got_mask, step = cache.find(0, h)
        bits_gpu = got_mask.bits.cpu().numpy()
        dense_gpu = mask_bits_to_dense(bits_gpu, m)
        k4 = bool((mask_bits_to_dense(ora.topk_select(S_dev[h], gamma), m) == dense_gpu).all())
        errs, errs_own = [], []
        for u in sample_blocks:
            lo, hi = u * block, min((u + 1) * block, n)
            ref_rows = ora.block_sparse_attention(rq, rk, rv, bits_ref, m, block, rows=(lo, hi))[lo:hi]
            got_rows = out[fwd[lo:hi].astype(np.int64), h]
            errs.append((np.abs(got_rows - ref_rows).max(), np.abs(ref_rows).max()))
            if (dense_gpu[u] != dense_ref[u]).any():
                own = ora.block_sparse_attention(rq, rk, rv, bits_gpu, m, block, rows=(lo, hi))[lo:hi]
            else:
                own = ref_rows
            errs_own.append((np.abs(got_rows - own).max(), np.abs(own).max()))
        res["heads"].append({
            "head": h,
            "score_err": float(np.abs(S_dev[h] - S_ref).max() / np.abs(S_ref).max()),
            "bit_agree": float((dense_gpu == dense_ref).mean()),
            "set_overlap": float((dense_gpu & dense_ref).sum() / dense_ref.sum()),
            "rows_equal": float((dense_gpu == dense_ref).all(1).mean()),
            "k4_exact": k4,
            "rows_sum_subs": float(np.abs(S_dev[h].sum(1) - block // sub).max()),
            "out_err": float(max(e for e, _ in errs) / max(r for _, r in errs)),
            "out_err_own": float(max(e for e, _ in errs_own) / max(r for _, r in errs_own)),
            "sampled_blocks": sample_blocks,
            "sparsity": float(stats.sparsity[h]),
            "last_update_step": int(step),
        })
    return res
