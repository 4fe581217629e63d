"""K3 tensor-core scorer (fp16x3 split, tcgen05) parity on the config shapes.

Tolerances: block scores max|S - S_ref| / max|S_ref| <= 1e-4
(expected ~1e-6 for an fp32-accurate scorer); mask agreement >= 99.5% of the
M^2 bits (expected 100%); masks bit-exact given identical scores (K4)."""
import numpy as np
import pytest

from oracle import mask_bits_to_dense, ora

from tests.golden.make_golden import CONFIGS, bf16_round

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dfs():
    import paper_2605_23445_b200 as m

    return m


def pooled_inputs(dims, d, heads, smooth=4.0):
    """bf16-rounded smooth fields in Hilbert order for `heads` heads (oracle-side arrays too)."""
    m = dfs()
    fwd = ora.hilbert3d_order(dims)
    qs, ks = [], []
    for h in range(heads):
        q, k, _ = (bf16_round(x) for x in ora.gen_video_field(dims, d, smooth, ora.derive_seed(1, [0, h])))
        qs.append(ora.apply_permutation(fwd, q))
        ks.append(ora.apply_permutation(fwd, k))
    return qs, ks


def gpu_scores(qs, ks, b, bs, generic=False):
    m = dfs()
    Q = torch.from_numpy(np.stack(qs, 1)).to(torch.bfloat16).cuda()
    K = torch.from_numpy(np.stack(ks, 1)).to(torch.bfloat16).cuda()
    h = m.default_handle()
    h.set_option(1, int(generic))
    try:
        return m.block_scores(Q, K, m.ScoringParams(b, bs)).cpu().numpy()
    finally:
        h.set_option(1, 0)


@pytest.mark.parametrize("cfg", ["T", "C", "W4"])
def test_scores_and_mask_agreement_vs_oracle(cfg):
    dims, H, d, gam = CONFIGS[cfg]
    b = 64 if cfg == "T" else 128
    qs, ks = pooled_inputs(dims, d, 2)
    S = gpu_scores(qs, ks, b, 16)
    for h in range(2):
        ref = ora.block_scores(qs[h], ks[h], b, 16)
        err = np.abs(S[h] - ref).max() / np.abs(ref).max()
        assert err <= 1e-4, (cfg, h, err)
        mm = ref.shape[0]
        want = mask_bits_to_dense(ora.topk_select(ref, gam), mm)
        got = mask_bits_to_dense(ora.topk_select(S[h], gam), mm)
        agree = (want == got).mean()
        assert agree >= 0.995, (cfg, h, agree)
        # K4 on the GPU scores is bit-exact with the oracle's selection on the same scores
        lut = dfs().topk_lut(torch.from_numpy(S[h]).cuda(), gam).cpu().numpy()
        dense = np.zeros_like(want)
        dense[np.arange(mm)[:, None], lut] = True
        assert (dense == got).all()


def test_scores_hunyuan_one_head_vs_oracle():
    dims, H, d, gam = CONFIGS["HY"]
    qs, ks = pooled_inputs(dims, d, 1)
    S = gpu_scores(qs, ks, 128, 16)[0]
    ref = ora.block_scores(qs[0], ks[0], 128, 16)
    err = np.abs(S - ref).max() / np.abs(ref).max()
    assert err <= 1e-4, err
    want = mask_bits_to_dense(ora.topk_select(ref, gam), 929)
    got = mask_bits_to_dense(ora.topk_select(S, gam), 929)
    assert (want == got).mean() >= 0.995
    assert np.allclose(S.sum(1), 8.0, rtol=1e-5)  # every row sums to subs (test_mask_builder.cpp:182-198)


def test_sm100_scorer_matches_generic_fp64_scorer_odd_geometry():
    """Both device scorers on ragged shapes and every supported B/B_s ratio."""
    rng = np.random.default_rng(0)
    for n, d, b, bs in [(1000, 64, 128, 16), (3001, 128, 128, 32), (777, 64, 64, 16), (4096, 128, 128, 8),
                        (300, 128, 64, 2)]:
        q = [bf16_round(rng.standard_normal((n, d)).astype(np.float32) * 3) for _ in range(2)]
        k = [bf16_round(rng.standard_normal((n, d)).astype(np.float32) * 3) for _ in range(2)]
        fast = gpu_scores(q, k, b, bs)
        slow = gpu_scores(q, k, b, bs, generic=True)
        for h in range(2):  # both device scorers against the C oracle (not CUDA against CUDA)
            ref = ora.block_scores(q[h], k[h], b, bs)
            assert np.abs(fast[h] - ref).max() / np.abs(ref).max() <= 1e-4, (n, d, b, bs, h)
            assert np.abs(slow[h] - ref).max() / np.abs(ref).max() <= 1e-9, (n, d, b, bs, h)


def test_scorer_extreme_magnitudes():
    """Per-head power-of-two scaling keeps both fp16 halves normal for tiny and huge inputs."""
    rng = np.random.default_rng(1)
    for scale in (1e-6, 8.0):  # logits std ~6 at 8.0; fp32 logits lose 1e-4 beyond ~|l| > 200
        # bf16-rounded: the device path takes bf16 activations, the oracle the same values upcast
        q = [bf16_round(rng.standard_normal((2048, 64)).astype(np.float32) * scale)]
        k = [bf16_round(rng.standard_normal((2048, 64)).astype(np.float32) * scale)]
        fast = gpu_scores(q, k, 128, 16)
        ref = ora.block_scores(q[0], k[0], 128, 16)
        assert np.abs(fast[0] - ref).max() / np.abs(ref).max() <= 1e-4, scale


def test_fuzz_pair_scorer_vs_fp64_scorer():
    """K3 runs as CTA pairs (two 128-row stripes of one head per pair): random head counts
    and lengths give odd stripe counts (a padded partner stripe), grids below 148 CTAs
    and every supported B/B_s ratio; scores must match the C oracle to 1e-4."""
    rng = np.random.default_rng(5)
    for trial in range(8):
        heads = int(rng.integers(1, 6))
        n = int(rng.integers(100, 6000))
        d = int(rng.choice([64, 128]))
        bs = int(rng.choice([8, 16, 32, 64]))
        q = [bf16_round(rng.standard_normal((n, d)).astype(np.float32) * 2) for _ in range(heads)]
        k = [bf16_round(rng.standard_normal((n, d)).astype(np.float32) * 2) for _ in range(heads)]
        fast = gpu_scores(q, k, 128, bs)
        for h in range(heads):  # against the C oracle's fp64 block_scores
            ref = ora.block_scores(q[h], k[h], 128, bs)
            err = np.abs(fast[h] - ref).max() / np.abs(ref).max()
            assert err <= 1e-4, (trial, heads, n, d, bs, h, err)
        assert np.allclose(fast.sum(-1), 128 // bs, rtol=1e-4)


def test_topk_tie_heavy_fuzz_bit_exact():
    """K4 (two 32-bit bisection phases) against the oracle's stable-sort selection on
    score matrices drawn from a handful of values (massive ties, equal high words) and on
    values that differ only in the low 32 bits of the double."""
    m = dfs()
    rng = np.random.default_rng(9)
    for mm in (7, 93, 256, 929, 1500):
        for kind in ("ties", "lowbits"):
            if kind == "ties":
                S = rng.choice(np.array([0.0, 1e-3, 0.25, 0.5, 1.0]), size=(mm, mm))
            else:
                base = np.float64(0.123456789).view(np.uint64)
                S = (base + rng.integers(0, 1 << 20, size=(mm, mm)).astype(np.uint64)).view(np.float64)
            for gam in (0.1, 0.37):
                lut = m.topk_lut(torch.from_numpy(S).cuda(), gam).cpu().numpy()
                got = np.zeros((mm, mm), bool)
                got[np.arange(mm)[:, None], lut] = True
                want = mask_bits_to_dense(ora.topk_select(S, gam), mm)
                assert (got == want).all(), (mm, kind, gam)


@pytest.mark.parametrize("jump", [4.0, 20.0, 60.0])
def test_scores_under_logit_jumps_across_key_tiles(jump):
    """The scorer's lazy row max (score_sm100.cu kLazy): a slice keeps the first key tile's max
    while its tile sums stay <= 2^16, and a later tile whose pooled logits jump by `jump` log2
    units (20 and 60 cross the test, 4 does not) raises it. Scores must still match the fp64
    oracle within 1e-4 and select the same masks."""
    rng = np.random.default_rng(11)
    n, d, b, bs = 8192, 128, 128, 16
    q = bf16_round((1.0 + 0.1 * rng.standard_normal((n, d))).astype(np.float32))
    k = 0.1 * rng.standard_normal((n, d)).astype(np.float32)
    # pooled logit of key tile 2 (pooled keys 256..383 = tokens 4096..6143) raised by `jump` log2 units
    c = jump / (d / d ** 0.5 * 1.4426950408889634)
    k[4096:6144] += c
    k = bf16_round(k)
    S = gpu_scores([q, q], [k, k], b, bs)
    ref = ora.block_scores(q, k, b, bs)
    for h in range(2):
        err = np.abs(S[h] - ref).max() / np.abs(ref).max()
        assert err <= 1e-4, (jump, h, err)
        mm = ref.shape[0]
        for gam in (0.1, 0.25):
            want = mask_bits_to_dense(ora.topk_select(ref, gam), mm)
            got = mask_bits_to_dense(ora.topk_select(S[h], gam), mm)
            assert (want == got).mean() >= 0.995, (jump, gam, h)
