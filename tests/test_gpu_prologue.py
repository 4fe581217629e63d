"""QK-norm + RoPE fused into K2 (dfs_qk_prologue; §8(f) row 1).

* the prologue alone (dfs_qk_prologue_apply) against a torch fp32 restatement of
  RMSNorm (x * w / sqrt(mean(x^2) + eps)) and RoPE (interleaved pairs and the
  rotate_half layout), within one bf16 rounding step;
* dfs.run_step(raw q, k, prologue=...) is bit-identical — outputs and masks, on
  update, mask-reuse and dense steps — to dfs.run_step on q, k transformed first
  (the fused pass changes where the transform runs, not what is computed).
"""
import math

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")

DIMS, H = (4, 16, 32), 3


def _tables(n, d, theta=10000.0):
    pos = torch.arange(n, dtype=torch.float64)
    inv = theta ** (-torch.arange(0, d // 2, dtype=torch.float64) * 2 / d)
    ang = pos[:, None] * inv[None, :]
    return ang.cos().float().cuda().contiguous(), ang.sin().float().cuda().contiguous()


def _torch_prologue(x, w, eps, rope, cos, sin):
    x = x.float()
    if w is not None:
        x = x * torch.rsqrt(x.pow(2).mean(-1, keepdim=True) + eps) * w
    if rope == "interleaved":
        a, b = x[..., 0::2], x[..., 1::2]
        c, s = cos[:, None, :], sin[:, None, :]
        x = torch.stack([a * c - b * s, a * s + b * c], -1).flatten(-2)
    elif rope == "half":
        h = x.shape[-1] // 2
        a, b = x[..., :h], x[..., h:]
        c, s = cos[:, None, :], sin[:, None, :]
        x = torch.cat([a * c - b * s, b * c + a * s], -1)
    return x.to(torch.bfloat16)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("rope", ["none", "interleaved", "half"])
@pytest.mark.parametrize("norm", [False, True])
def test_prologue_matches_torch(d, rope, norm):
    import paper_2605_23445_b200 as dfs

    n = math.prod(DIMS)
    g = torch.Generator().manual_seed(d)
    x = (torch.randn(n, H, d, generator=g) * 3).to(torch.bfloat16).cuda()
    w = (torch.rand(d, generator=g) + 0.5).cuda() if norm else None
    cos, sin = _tables(n, d)
    pro = dfs.QkPrologue(q_norm_weight=w, eps=1e-6, rope=rope, rope_cos=cos, rope_sin=sin)
    got = pro.apply(x, "q").float()
    want = _torch_prologue(x, w, 1e-6, rope, cos, sin).float()
    # fp32 math in a different order: at most one bf16 rounding step apart
    assert ((got - want).abs() <= want.abs() * 2 ** -7 + 1e-6).all()


@pytest.mark.parametrize("d", [64, 128])
def test_run_step_with_prologue_equals_pretransformed(d):
    import paper_2605_23445_b200 as dfs

    n = math.prod(DIMS)
    g = torch.Generator().manual_seed(11 + d)
    q, k, v = ((torch.randn(n, H, d, generator=g) * 2).to(torch.bfloat16).cuda() for _ in range(3))
    cos, sin = _tables(n, d)
    pro = dfs.QkPrologue(q_norm_weight=(torch.rand(d, generator=g) + 0.5).cuda(),
                         k_norm_weight=(torch.rand(d, generator=g) + 0.5).cuda(), eps=1e-6, rope="half",
                         rope_cos=cos, rope_sin=sin)
    qt, kt = pro.apply(q, "q"), pro.apply(k, "k")
    sched = dfs.SparsitySchedule(total_steps=4, warmup_fraction=0.25, phase_budgets=(0.25,), phase_fraction=0.75,
                                 update_interval=2)
    params = dfs.ScoringParams(128, 16)
    c1, c2 = dfs.MaskCache(), dfs.MaskCache()
    for step in range(4):  # dense, update, reuse, update
        o1, s1 = dfs.run_step(q, k, v, DIMS, params, sched, c1, 0, step, prologue=pro)
        o2, s2 = dfs.run_step(qt, kt, v, DIMS, params, sched, c2, 0, step)
        torch.cuda.synchronize()
        assert s1.dense == s2.dense and s1.mask_updated == s2.mask_updated
        assert torch.equal(o1, o2), step
        if not s1.dense:
            for h in range(H):
                assert torch.equal(c1.find(0, h)[0].bits, c2.find(0, h)[0].bits)


def test_prologue_nonfinite_is_refused():
    import paper_2605_23445_b200 as dfs

    n, d = math.prod(DIMS), 128
    q = torch.randn(n, H, d).to(torch.bfloat16).cuda()
    bad = q.clone()
    bad[5, 1, 3] = float("inf")
    pro = dfs.QkPrologue(q_norm_weight=torch.ones(d).cuda())
    sched = dfs.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(0.25,), phase_fraction=1.0,
                                 update_interval=1)
    cache = dfs.MaskCache()
    with pytest.raises(ValueError):
        dfs.run_step(bad, q, q, DIMS, dfs.ScoringParams(128, 16), sched, cache, 0, 0, prologue=pro)
    assert cache.size() == 0
