"""GPU parity: the CUDA path (through the C ABI) against the oracle and the
reference-generated golden fixtures. Tolerances:
  * permutations, masks given identical scores: bit-exact;
  * geometry-generic fp64 scorer: |S - S_ref| <= 1e-9 relative, masks equal;
  * fp32 attention (drop-in Matrix path): max abs err <= 1e-5 (the reference's
    own test tolerance, test_attention.cpp:124-200);
  * bf16 I/O attention: max|O - O_ref| / max|O_ref| <= 2e-2 per head.
"""
import numpy as np
import pytest

from oracle import dense_to_mask_bits, mask_bits_to_dense, ora

from tests.golden.make_golden import CONFIGS, bf16_round

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dfs():
    import paper_2605_23445_b200 as m

    return m


def cu(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    return t if dtype is None else t.to(dtype)


def host(t):
    return t.detach().cpu().numpy()


# ------------------------------------------------------------------ K1 -----

def test_hilbert_bit_exact_all_configs(golden):
    g = golden("perms")
    for name, (dims, _, _, _) in CONFIGS.items():
        fwd = host(dfs().hilbert3d_order(dims).forward).astype(np.uint32)
        assert (fwd == ora.hilbert3d_order(dims)).all(), name
        assert (fwd[:256] == g[f"{name}_head"]).all() and (fwd[-256:] == g[f"{name}_tail"]).all()


def test_all_orderings_bit_exact(golden):
    g = golden("perms")
    for key, want in g.items():
        if not key.startswith("order_"):
            continue
        _, o, dims = key.split("_")
        f, h, w = (int(x) for x in dims.split("x"))
        assert (host(dfs().order_tokens(o, (f, h, w)).forward).astype(np.uint32) == want).all(), key
    rng = np.random.default_rng(2024)  # test_curve.cpp:138-151
    for _ in range(20):
        dims = tuple(int(x) for x in rng.integers(1, 65, size=3))
        for o in ("raster", "hilbert2d", "block3d", "hilbert3d"):
            got = host(dfs().order_tokens(o, dims).forward).astype(np.uint32)
            assert (got == ora.order_tokens(o, dims)).all(), (o, dims)


def test_invert_validate_and_round_trip():
    m = dfs()
    perm = m.hilbert3d_order((33, 45, 80))
    inv = m.invert_permutation(perm)
    assert (host(inv.forward).astype(np.uint32) == ora.invert_permutation(host(perm.forward).astype(np.uint32))).all()
    m.validate_permutation(perm.forward)
    bad = perm.forward.clone()
    bad[5] = bad[6]
    with pytest.raises(ValueError):
        m.validate_permutation(bad)
    # apply(invert(p), apply(p, x)) == x bit-exactly (acceptance criterion 4), batched bf16 heads
    x = torch.randn(perm.size(), 24, 128, device="cuda").to(torch.bfloat16)
    y = m.apply_permutation(perm, x)
    assert torch.equal(y[7], x[int(perm.forward[7])])
    assert torch.equal(m.apply_permutation(inv, y), x)
    assert torch.equal(m.unpermute(perm, y), x)
    # fp32 single head, odd d (scalar path)
    x2 = torch.randn(perm.size(), 5, device="cuda")
    assert torch.equal(m.unpermute(perm, m.apply_permutation(perm, x2)), x2)
    with pytest.raises(ValueError):
        m.apply_permutation(perm, x2[:-1])


# ------------------------------------------------------------------ K2 -----

def test_mean_pool_bit_exact():
    rng = np.random.default_rng(5)
    for n, d, pool in [(6, 3, 2), (3, 1, 2), (100, 64, 16), (17550, 64, 16), (1000, 128, 16), (37, 8, 5)]:
        x = rng.standard_normal((n, d)).astype(np.float32)
        got = host(dfs().mean_pool(cu(x), pool))
        assert (got == ora.mean_pool(x, pool)).all(), (n, d, pool)
        xb = bf16_round(x)
        got = host(dfs().mean_pool(cu(xb).to(torch.bfloat16), pool))
        assert (got == ora.mean_pool(xb, pool)).all()
    with pytest.raises(ValueError):
        dfs().mean_pool(cu(np.zeros((4, 2), np.float32)), 0)


# -------------------------------------------------------------- K3 / K4 -----

def test_topk_bit_exact_given_reference_scores(golden):
    g = golden("kats")
    for gam in (0.02, 0.1, 0.37, 0.5, 1.0):  # tie-heavy rows
        mask = dfs().topk_select(cu(g["ties"]), gam, 16)
        assert (host(mask.bits) == g[f"ties_{gam}"]).all(), gam
    c = golden("cogvideo_h0")
    mask = dfs().topk_select(cu(c["S"]), 0.2, 128)
    assert (host(mask.bits) == c["bits"]).all()
    # test_mask_builder.cpp:210-243 examples
    S = np.array([[0.4, 0.1, 0.4, 0.1], [0.4, 0.4, 0.1, 0.1], [0.25] * 4, [4, 3, 2, 1]], np.float64)
    lut = host(dfs().topk_lut(cu(S), 0.5))
    assert lut.tolist() == [[0, 2], [0, 1], [0, 1], [0, 1]]
    lut1 = host(dfs().topk_lut(cu(S), 0.25))
    assert lut1[:, 0].tolist() == [0, 0, 0, 0]
    # random rows with injected ties vs the oracle, batched heads
    rng = np.random.default_rng(11)
    for m_ in (1, 7, 64, 929, 2000):
        s = np.round(rng.random((3, m_, m_)) * 50) / 50
        for gam in (0.05, 0.1, 0.5):
            got = host(dfs().topk_lut(cu(s), gam))
            k = ora.topk_count(gam, m_)
            for h in range(3):
                lut_o = np.zeros((m_, k), np.int32)
                bits = np.zeros((m_ * m_ + 7) // 8, np.uint8)
                import ctypes as C
                ora.lib.oracle_topk_select.restype = C.c_int
                ora.lib.oracle_topk_select(np.ascontiguousarray(s[h]).ctypes.data_as(C.c_void_p), C.c_int64(m_),
                                           C.c_double(gam), bits.ctypes.data_as(C.c_void_p),
                                           lut_o.ctypes.data_as(C.c_void_p))
                assert (got[h] == lut_o).all(), (m_, gam, h)


class generic_scorer:
    """Route block scoring through the fp64 geometry-generic kernel (handle option)."""

    def __enter__(self):
        dfs().default_handle().set_option(1, 1)

    def __exit__(self, *exc):
        dfs().default_handle().set_option(1, 0)


def test_scores_and_masks_small_cases(golden):
    """fp64 generic scorer: 1e-9 and bit-exact masks; tcgen05 scorer (d in {64,128}):
    1e-4 and >= 99.5% mask agreement."""
    g = golden("kats")
    for i in g["cases"]:
        n, d, b, bs, gam = g[f"c{i}_meta"]
        n, d, b, bs = int(n), int(d), int(b), int(bs)
        q, k = g[f"c{i}_q"], g[f"c{i}_k"]
        ref = g[f"c{i}_S"]
        with generic_scorer():
            S = host(dfs().block_scores(cu(q), cu(k), dfs().ScoringParams(b, bs)))
            assert np.abs(S - ref).max() <= 1e-9 * max(1.0, np.abs(ref).max()), i
            mask = dfs().build_mask(cu(q), cu(k), dfs().ScoringParams(b, bs), float(gam))
            assert (host(mask.bits) == g[f"c{i}_bits"]).all(), i
        S = host(dfs().block_scores(cu(q), cu(k), dfs().ScoringParams(b, bs)))
        assert np.abs(S - ref).max() <= 1e-4 * np.abs(ref).max(), i
        mm = ref.shape[0]
        mask = dfs().build_mask(cu(q), cu(k), dfs().ScoringParams(b, bs), float(gam))
        agree = (mask_bits_to_dense(host(mask.bits), mm) == mask_bits_to_dense(g[f"c{i}_bits"], mm)).mean()
        assert agree >= 0.995, (i, agree)


def test_tiny_config_scores(golden):
    g = golden("tiny")
    for h in range(2):
        rq = ora.apply_permutation(g["fwd"], g[f"q{h}"])
        rk = ora.apply_permutation(g["fwd"], g[f"k{h}"])
        with generic_scorer():
            S = host(dfs().block_scores(cu(rq), cu(rk), dfs().ScoringParams(64, 16)))
        assert np.abs(S - g[f"S{h}"]).max() <= 1e-9
        mask = dfs().topk_select(cu(S), 0.5, 64)
        assert (host(mask.bits) == g[f"bits{h}"]).all()
        S2 = host(dfs().block_scores(cu(rq), cu(rk), dfs().ScoringParams(64, 16)))
        assert np.abs(S2 - g[f"S{h}"]).max() <= 1e-4 * np.abs(g[f"S{h}"]).max()
        assert (host(dfs().topk_select(cu(S2), 0.5, 64).bits) == g[f"bits{h}"]).all()


# ------------------------------------------------------------------ K5 -----

def test_attention_fp32_matches_reference_kats(golden):
    g = golden("kats")
    for i in g["cases"]:
        n, d, b, bs, gam = g[f"c{i}_meta"]
        n, d, b = int(n), int(d), int(b)
        q, k, v = (cu(g[f"c{i}_{x}"]) for x in "qkv")
        m = -(-n // b)
        mask = dfs().BlockMask(cu(g[f"c{i}_bits"]), m, b)
        out = host(dfs().block_sparse_attention(q, k, v, mask))
        assert np.abs(out - g[f"c{i}_o"]).max() <= 1e-5, i
    out = host(dfs().full_attention_output(cu(g["x_q"]), cu(g["x_k"]), cu(g["x_v"])))
    assert np.abs(out - g["x_o"]).max() <= 1e-5


def test_attention_reference_semantics():
    m = dfs()
    rng = np.random.default_rng(23)
    # all-ones mask == dense (test_attention.cpp:124-138, acceptance criterion 1)
    for _ in range(20):
        n, d, b = int(rng.integers(1, 300)), int(rng.integers(1, 64)), int(rng.integers(1, 129))
        q, k, v = (rng.standard_normal((n, d)).astype(np.float32) for _ in range(3))
        mm = -(-n // b)
        full = m.BlockMask.full(mm, b, True)
        sparse = host(m.block_sparse_attention(cu(q), cu(k), cu(v), full))
        dense = ora.full_attention_output(q, k, v)
        assert np.abs(sparse - dense).max() <= 1e-5
    # diagonal mask == per-block attention (test_attention.cpp:140-164)
    b, mb, d = 4, 3, 5
    q, k, v = (rng.standard_normal((b * mb, d)).astype(np.float32) for _ in range(3))
    diag = m.BlockMask.from_dense(torch.eye(mb, dtype=torch.bool), b)
    out = host(m.block_sparse_attention(cu(q), cu(k), cu(v), diag))
    for u in range(mb):
        sl = slice(u * b, (u + 1) * b)
        assert np.abs(out[sl] - ora.full_attention_output(q[sl], k[sl], v[sl])).max() <= 1e-5
    # padded keys excluded / padded queries not produced (test_attention.cpp:190-200)
    q, k, v = (rng.standard_normal((5, 3)).astype(np.float32) for _ in range(3))
    out = host(m.block_sparse_attention(cu(q), cu(k), cu(v), m.BlockMask.full(2, 4, True)))
    assert out.shape == (5, 3) and np.abs(out - ora.full_attention_output(q, k, v)).max() <= 1e-5
    # errors (test_attention.cpp:202-218)
    q4 = cu(rng.standard_normal((4, 2)).astype(np.float32))
    one_row = m.BlockMask.from_dense(torch.tensor([[True, False], [False, False]]), 2)
    with pytest.raises(ValueError):
        m.block_sparse_attention(q4, q4, q4, one_row)
    q8 = cu(np.zeros((8, 2), np.float32))
    with pytest.raises(ValueError):
        m.block_sparse_attention(q8, q8, q8, m.BlockMask.full(3, 2, True))
    bad = q4.clone()
    bad[0, 0] = float("nan")
    with pytest.raises(ValueError):
        m.block_sparse_attention(bad, q4, q4, m.BlockMask.full(2, 2, True))


def _rel_err(o, ref):
    return float(np.abs(o - ref).max() / max(np.abs(ref).max(), 1e-30))


def test_attention_bf16_cogvideo_head0(golden):
    """bf16 I/O at the C shape, oracle rows from the reference (tolerance 2e-2 per head)."""
    c = golden("cogvideo_h0")
    dims, _, d, gam = CONFIGS["C"]
    s = ora.derive_seed(1, [0, 0])
    q, k, v = (bf16_round(x) for x in ora.gen_video_field(dims, d, 4.0, s))
    fwd = ora.hilbert3d_order(dims)
    rq, rk, rv = (ora.apply_permutation(fwd, x) for x in (q, k, v))
    m_ = c["S"].shape[0]
    mask = dfs().BlockMask(cu(c["bits"]), m_, 128)
    for generic in (True, False):
        out = host(dfs().block_sparse_attention(cu(rq, torch.bfloat16), cu(rk, torch.bfloat16),
                                                cu(rv, torch.bfloat16), mask, force_generic=generic).float())
        rows = c["rows"]
        assert _rel_err(out[rows], c["o_rows"]) <= 2e-2


# ------------------------------------------------------- step / cache -------

def _tiny_heads():
    dims, H, d, gam = CONFIGS["T"]
    qs, ks, vs = [], [], []
    for h in range(H):
        q, k, v = (bf16_round(x) for x in ora.gen_video_field(dims, d, 4.0, ora.derive_seed(1, [0, h])))
        qs.append(q), ks.append(k), vs.append(v)
    return dims, H, d, gam, np.stack(qs, 1), np.stack(ks, 1), np.stack(vs, 1)


def test_run_step_tiny_config_matches_reference(golden):
    """Config T through the batched Alg. 1 step ([N, H, d] bf16 raster in/out)."""
    g = golden("tiny")
    m = dfs()
    dims, H, d, gam, Q, K, V = _tiny_heads()
    sched = m.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(gam,), phase_fraction=1.0,
                               update_interval=1)
    cache = m.MaskCache()
    out, st = m.run_step(cu(Q, torch.bfloat16), cu(K, torch.bfloat16), cu(V, torch.bfloat16), dims,
                         m.ScoringParams(64, 16), sched, cache, layer=0, step=0)
    assert not st.dense and all(st.mask_updated)
    out = host(out.float())
    fwd = g["fwd"]
    inv = ora.invert_permutation(fwd)
    for h in range(H):
        found = cache.find(0, h)
        assert found is not None and found[1] == 0
        assert (host(found[0].bits) == g[f"bits{h}"]).all()
        ref_raster = ora.apply_permutation(inv, g[f"o{h}"])
        assert _rel_err(out[:, h], ref_raster) <= 2e-2
        assert st.sparsity[h] == 0.5


def test_dense_step_and_phase_lag():
    """Warmup steps are dense in raster order; a cached mask keeps the K of its
    update step across a phase change (scheduler.cpp:85-89, test_cli.cpp:279-283)."""
    m = dfs()
    dims, H, d, gam, Q, K, V = _tiny_heads()
    q, k, v = (cu(x, torch.bfloat16) for x in (Q, K, V))
    sched = m.SparsitySchedule(total_steps=10, warmup_fraction=0.2, phase_budgets=(0.5, 0.25), phase_fraction=0.4,
                               update_interval=3)
    cache = m.MaskCache()
    params = m.ScoringParams(64, 16)
    out, st = m.run_step(q, k, v, dims, params, sched, cache, 0, 0)
    assert st.dense and cache.empty()
    dense_ref = np.stack([ora.full_attention_output(Q[:, h], K[:, h], V[:, h]) for h in range(H)], 1)
    assert _rel_err(host(out.float()), dense_ref) <= 2e-2
    flags = []
    for step in range(2, 10):
        _, st = m.run_step(q, k, v, dims, params, sched, cache, 0, step)
        flags.append((step, st.mask_updated[0], st.budget, st.sparsity[0]))
    # updates at sparse steps 2, 5, 8; phases: 2-5 -> 0.5, 6-9 -> 0.25
    assert [f[1] for f in flags] == [s in (2, 5, 8) for s in range(2, 10)]
    # steps 6 and 7 reuse the 0.5-budget mask from step 5: sparsity 0.5, not 0.75
    assert [f[3] for f in flags if f[0] in (6, 7)] == [0.5, 0.5]
    assert flags[-2][3] == 0.75  # step 8 refreshes at 0.25 -> K=1 of M=4


def test_mask_cache_store_find_roundtrip():
    m = dfs()
    cache = m.MaskCache()
    assert cache.empty() and not cache.contains(0, 0)
    rng = np.random.default_rng(9)
    dense = rng.random((7, 7)) < 0.4
    dense[np.arange(7), np.arange(7)] = True
    mask = m.BlockMask.from_dense(torch.from_numpy(dense), 16)
    cache.store(2, 3, mask, 12)
    assert cache.contains(2, 3) and not cache.contains(2, 0) and cache.size() == 1
    got, step = cache.find(2, 3)
    assert step == 12 and torch.equal(got.bits.cpu(), mask.bits.cpu())
    dense2 = np.eye(7, dtype=bool)
    cache.store(2, 0, m.BlockMask.from_dense(torch.from_numpy(dense2), 16), 24)
    got0, s0 = cache.find(2, 0)
    got3, s3 = cache.find(2, 3)
    assert (got0.to_dense().numpy() == dense2).all() and (got3.to_dense().numpy() == dense).all()
    assert (s0, s3) == (24, 12) and cache.size() == 2
    cache.clear()
    assert cache.empty()


def test_trajectory_masks_match_reference(golden):
    """cmd_run-style trajectory (commands.cpp:221-319) through the batched device step on
    the reference's OWN fp32 inputs (dfs.run_step with fp32 [N, H, d]: the compatibility
    kernels, fp64 softmax arithmetic): every (step, layer, head) dense / update flag and
    every cached mask is bit-identical to the reference's, and the sparse outputs match the
    oracle's attention under that mask at the reference's 1e-5 tolerance."""
    t = golden("trajectory")
    f, h_, w, d, L, H, T, b, bs = (int(x) for x in t["meta"])
    m = dfs()
    budgets = tuple(float(x) for x in t["budgets"])
    sched = m.SparsitySchedule(total_steps=T, warmup_fraction=0.2, phase_budgets=budgets, phase_fraction=0.4,
                               update_interval=3)
    cache = m.MaskCache()
    params = m.ScoringParams(b, bs)
    n = f * h_ * w
    mm = -(-n // b)
    fwd = ora.hilbert3d_order((f, h_, w))
    inv = ora.invert_permutation(fwd)
    dense_layers = set(int(x) for x in t["dense_layers"])
    for step in range(T):
        for layer in range(L):
            Qs, Ks, Vs = [], [], []
            for head in range(H):
                seed = ora.derive_seed(1, [layer * H + head])
                q, k, v = ora.trajectory_at((f, h_, w), d, 4.0, seed, T, 2.0, 0.0, step)
                Qs.append(q), Ks.append(k), Vs.append(v)
            Q, K, V = (np.stack(x, 1) for x in (Qs, Ks, Vs))
            out, st = m.run_step(cu(Q), cu(K), cu(V), (f, h_, w), params, sched, cache, layer, step,
                                 force_dense=layer in dense_layers)
            out = host(out)
            for head in range(H):
                row = step * L * H + layer * H + head
                flags = int(t["flags"][row])
                assert st.dense == bool(flags & 1), (step, layer, head)
                assert st.budget == t["budget"][row] and st.sparsity[head] == t["sparsity"][row], (step, layer, head)
                if layer == 0 and head == 0:  # the reference's own output of (layer 0, head 0), every step
                    assert np.abs(out[:, 0] - t["out00"][step]).max() <= 1e-5, step
                if st.dense:
                    continue
                assert st.mask_updated[head] == bool(flags & 2), (step, layer, head)
                got, ls = cache.find(layer, head)
                if st.mask_updated[head]:
                    assert ls == step
                    assert (host(got.bits) == t["masks"][row]).all(), (step, layer, head)
                rq, rk, rv = (ora.apply_permutation(fwd, x[:, head]) for x in (Q, K, V))
                ref = ora.apply_permutation(inv, ora.block_sparse_attention(rq, rk, rv, host(got.bits), mm, b))
                assert np.abs(out[:, head] - ref).max() <= 1e-5, (step, layer, head)


@pytest.mark.parametrize("d", [96, 128])
def test_run_step_generic_and_tcgen05_paths(d):
    """run_step at B = 128 on a ragged lattice: d = 96 is refused by default and, opted in,
    takes the geometry-generic kernels (fp64 scorer, SIMT attention with the gathered
    query rows); d = 128 the tcgen05 ones.
    Masks: bit-exact vs the oracle for the fp64 scorer, >= 99.5 % agreement for the
    fp16x3 one; outputs vs the oracle's attention under the device's own mask."""
    m = dfs()
    dims, H, gam, b, bs = (3, 16, 61), 2, 0.25, 128, 16
    n = int(np.prod(dims))
    qs, ks, vs = [], [], []
    for h in range(H):
        q, k, v = (bf16_round(x) for x in ora.gen_video_field(dims, d, 4.0, ora.derive_seed(3, [0, h])))
        qs.append(q), ks.append(k), vs.append(v)
    Q, K, V = (torch.from_numpy(np.stack(x, 1)).to(torch.bfloat16).cuda() for x in (qs, ks, vs))
    sched = m.SparsitySchedule(total_steps=1, warmup_fraction=0.0, phase_budgets=(gam,), phase_fraction=1.0,
                               update_interval=1)
    cache = m.MaskCache()
    if d == 96:  # outside the tcgen05 contract: refused up front (nothing cached), unless opted in
        with pytest.raises(m._capi.UnsupportedGeometry):
            m.run_step(Q, K, V, dims, m.ScoringParams(b, bs), sched, cache, layer=0, step=0)
        assert cache.size() == 0
        cache.handle.set_option(2, 1)  # DFS_OPT_GENERIC_ATTN
    out, st = m.run_step(Q, K, V, dims, m.ScoringParams(b, bs), sched, cache, layer=0, step=0)
    out = host(out.float())
    fwd = ora.hilbert3d_order(dims)
    inv = ora.invert_permutation(fwd)
    mm = -(-n // b)
    for h in range(H):
        rq, rk, rv = (ora.apply_permutation(fwd, x[h]) for x in (qs, ks, vs))
        want = mask_bits_to_dense(ora.build_mask(rq, rk, b, bs, gam), mm)
        bits = host(cache.find(0, h)[0].bits)
        got = mask_bits_to_dense(bits, mm)
        if d == 96:
            assert (got == want).all()
        else:
            assert (got == want).mean() >= 0.995
        ref = ora.apply_permutation(inv, ora.block_sparse_attention(rq, rk, rv, bits, mm, b))
        assert _rel_err(out[:, h], ref) <= 2e-2, (d, h)


@pytest.mark.parametrize("which", ["q", "k", "v"])
def test_run_step_nonfinite_refused_by_default(which):
    """attention.cpp:19-20: non-finite input is an error — by default, on dense, update and
    reuse steps — with the reference's ordering: a non-finite q or k raises from build_mask
    (attention_scores) before the mask is stored, a non-finite v from block_sparse_attention
    AFTER build_mask stored it (scheduler.cpp:113-122); no output is written either way."""
    m = dfs()
    dims, H, d, b, bs = (4, 16, 32), 2, 128, 128, 16
    n = int(np.prod(dims))
    g = torch.Generator().manual_seed(3)
    q, k, v = (torch.randn(n, H, d, generator=g).to(torch.bfloat16).cuda() for _ in range(3))
    sched = m.SparsitySchedule(total_steps=4, warmup_fraction=0.25, phase_budgets=(0.25,), phase_fraction=0.75,
                               update_interval=2)
    params = m.ScoringParams(b, bs)
    cache = m.MaskCache()
    bad = {"q": q, "k": k, "v": v}
    t = bad[which].clone()
    t[n // 2, 1, 5] = float("nan")
    bad[which] = t
    out = torch.zeros_like(q)
    with pytest.raises(ValueError):  # dense step
        m.run_step(bad["q"], bad["k"], bad["v"], dims, params, sched, cache, 0, 0, out=out)
    with pytest.raises(ValueError):  # first sparse step: nothing cached yet
        m.run_step(bad["q"], bad["k"], bad["v"], dims, params, sched, cache, 0, 1, out=out)
    assert cache.size() == (H if which == "v" else 0)
    assert not out.any()  # no output written
    m.run_step(q, k, v, dims, params, sched, cache, 0, 1)
    before = [cache.find(0, h)[0].bits.clone() for h in range(H)]
    with pytest.raises(ValueError):  # reuse step
        m.run_step(bad["q"], bad["k"], bad["v"], dims, params, sched, cache, 0, 2, out=out)
    for h in range(H):
        assert cache.find(0, h)[1] == 1 and torch.equal(cache.find(0, h)[0].bits, before[h])
    with pytest.raises(ValueError):  # update step: only a bad v lets the new mask be stored
        m.run_step(bad["q"], bad["k"], bad["v"], dims, params, sched, cache, 0, 3, out=out)
    for h in range(H):
        assert cache.find(0, h)[1] == (3 if which == "v" else 1)
    assert not out.any()
