"""Streaming attention recall (recall_sm100.cu) vs the reference's definition,
attention_recall(attention_scores(rq, rk), mask) (attention.cpp:105-123,175-190,
scheduler.cpp:129-131), restated in fp64 numpy at sizes where A fits; and at the
HunyuanVideo shape, past the reference's 4096-row cap, where the reference refuses."""
import numpy as np
import pytest

from oracle import mask_bits_to_dense, ora

from tests.golden.make_golden import bf16_round

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dfs():
    import paper_2605_23445_b200 as m

    return m


def recall_ref(rq, rk, dense_mask, b):
    a = rq.astype(np.float64) @ rk.astype(np.float64).T / np.sqrt(rq.shape[1])
    a = np.exp(a - a.max(1, keepdims=True))
    a /= a.sum(1, keepdims=True)
    a = a.astype(np.float32).astype(np.float64)  # A is stored in fp32 (attention.cpp:120)
    n = rq.shape[0]
    m = np.kron(dense_mask, np.ones((b, b), bool))[:n, :n]
    return float((a * m).sum() / a.sum())


@pytest.mark.parametrize("d", [64, 128])
def test_run_step_recall_matches_reference_definition(d):
    m = dfs()
    dims, H, gam, b, bs = (4, 16, 50), 2, 0.25, 128, 16
    n = int(np.prod(dims))
    qs, ks, vs = [], [], []
    for h in range(H):
        q, k, v = (bf16_round(x) for x in ora.gen_video_field(dims, d, 4.0, ora.derive_seed(9, [0, h])))
        qs.append(q), ks.append(k), vs.append(v)
    Q, K, V = (torch.from_numpy(np.stack(x, 1)).to(torch.bfloat16).cuda() for x in (qs, ks, vs))
    sched = m.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(gam,), phase_fraction=1.0,
                               update_interval=1)
    cache = m.MaskCache()
    _, st = m.run_step(Q, K, V, dims, m.ScoringParams(b, bs), sched, cache, layer=0, step=0, record_recall=True)
    fwd = ora.hilbert3d_order(dims)
    mm = -(-n // b)
    for h in range(H):
        dense = mask_bits_to_dense(cache.find(0, h)[0].bits.cpu().numpy(), mm)
        want = recall_ref(ora.apply_permutation(fwd, qs[h]), ora.apply_permutation(fwd, ks[h]), dense, b)
        assert abs(st.recall[h] - want) <= 1e-4 * max(want, 1e-3), (h, st.recall[h], want)
        assert 0.25 <= st.recall[h] <= 1.0  # keeps at least the budget's share (top-K by mass)


def test_recall_full_mask_is_one_and_dense_step_reports_one():
    m = dfs()
    H, n, d = 2, 1000, 128
    g = torch.Generator(device="cuda").manual_seed(3)
    q, k = (torch.randn(H, n, d, generator=g, device="cuda").bfloat16() for _ in range(2))
    mq = -(-n // 128)
    lut = torch.arange(mq, dtype=torch.int32, device="cuda").repeat(H * mq)
    ptr = m.ops.lut_row_ptr(H, mq, mq)
    rec = m.block_recall(q, k, ptr, lut)
    assert all(abs(r - 1.0) < 1e-6 for r in rec), rec


def test_recall_at_hunyuan_shape_past_the_dense_cap():
    """N = 118,800 (the reference's attention_scores refuses > 4096 rows): recall of the
    top-10% masks of smooth fields is well above the 10% budget and below 1."""
    from bench import smooth_fields

    m = dfs()
    dims, H, d = (33, 45, 80), 4, 128
    q, k, v = smooth_fields(dims, H, d, seed=2, device=torch.device("cuda"))
    sched = m.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(0.1,), phase_fraction=1.0,
                               update_interval=1)
    _, st = m.run_step(q, k, v, dims, m.ScoringParams(128, 16), sched, m.MaskCache(), layer=0, step=0,
                       record_recall=True)
    assert all(0.1 < r < 1.0 for r in st.recall), st.recall
