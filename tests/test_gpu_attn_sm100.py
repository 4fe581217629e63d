"""K5 tcgen05 kernel parity: against the oracle (fp64, the reference's
arithmetic) on sampled rows, and against the geometry-generic SIMT kernel on
full tensors. bf16 I/O tolerance: max|O - O_ref| / max|O_ref| <= 2e-2 per head
(SURVEY.md §8(d)); observed errors are ~3e-3."""
import numpy as np
import pytest

from oracle import ora

from tests.golden.make_golden import bf16_round

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")


def dfs():
    import paper_2605_23445_b200 as m

    return m


def rel(o, ref):
    return float((o - ref).abs().max() / ref.abs().max().clamp_min(1e-30))


def random_lut(h, mq, mk, k, gen):
    idx = torch.stack([torch.stack([torch.randperm(mk, generator=gen)[:k].sort().values for _ in range(mq)])
                       for _ in range(h)])
    return idx.to(torch.int32)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("n,k", [(128, 1), (1000, 3), (4096 + 77, 7), (17550, 28)])
def test_sm100_matches_generic_hnd_lut(d, n, k):
    m = dfs()
    gen = torch.Generator().manual_seed(n * d + k)
    h = 3
    q, kk, v = (torch.randn(h, n, d, generator=gen).to(torch.bfloat16).cuda() for _ in range(3))
    mq = -(-n // 128)
    k = min(k, mq)
    lut = random_lut(h, mq, mq, k, gen).cuda()
    ptr = m.ops.lut_row_ptr(h, mq, k)
    o_fast = m.sparse_attention_csr(q, kk, v, ptr, lut.reshape(-1), 128)
    o_ref = m.sparse_attention_csr(q, kk, v, ptr, lut.reshape(-1), 128, force_generic=True)
    torch.cuda.synchronize()
    for hh in range(h):
        assert rel(o_fast[hh].float(), o_ref[hh].float()) <= 1e-2, hh


@pytest.mark.parametrize("d", [64, 128])
def test_sm100_dense_nhd_and_cross_attention(d):
    m = dfs()
    gen = torch.Generator().manual_seed(7 + d)
    h, nq, nk = 2, 777, 1500
    q = torch.randn(nq, h, d, generator=gen).to(torch.bfloat16).cuda()
    k = torch.randn(nk, h, d, generator=gen).to(torch.bfloat16).cuda()
    v = torch.randn(nk, h, d, generator=gen).to(torch.bfloat16).cuda()
    o = m.full_attention_output(q, k, v)  # Nq != Nk through K5 with a full mask
    og = m.full_attention_output(q, k, v, force_generic=True)
    assert rel(o.float(), og.float()) <= 1e-2
    qf, kf, vf = (x.float().cpu().numpy() for x in (q, k, v))
    for hh in range(h):
        ref = ora.full_attention_output(qf[:, hh], kf[:, hh], vf[:, hh], rows=(0, 200))
        got = o[:200, hh].float().cpu()
        assert rel(got, torch.from_numpy(ref[:200])) <= 2e-2


def test_sm100_scatter_epilogue_matches_unpermute():
    """out_rows fuses the inverse permutation (scheduler.cpp:134) into K5's epilogue."""
    m = dfs()
    dims = (13, 30, 45)
    n, h, d = 13 * 30 * 45, 4, 64
    gen = torch.Generator().manual_seed(3)
    q, k, v = (torch.randn(h, n, d, generator=gen).to(torch.bfloat16).cuda() for _ in range(3))
    perm = m.hilbert3d_order(dims)
    mq = -(-n // 128)
    lut = random_lut(h, mq, mq, 28, gen).cuda()
    ptr = m.ops.lut_row_ptr(h, mq, 28)
    o_hnd = m.sparse_attention_csr(q, k, v, ptr, lut.reshape(-1), 128)           # reordered [H, N, d]
    o_nhd = m.sparse_attention_csr(q, k, v, ptr, lut.reshape(-1), 128, out_layout=0,
                                   out_rows=perm.forward)                         # raster [N, H, d]
    want = m.unpermute(perm, o_hnd.transpose(0, 1).contiguous())
    assert torch.equal(o_nhd, want)


@pytest.mark.slow
def test_sm100_hunyuan_two_heads_vs_oracle_rows():
    """HY geometry (118,800 tokens, d=128, K=93 of 929): smooth inputs, real
    top-K masks from the GPU scorer, sampled rows against the fp64 oracle."""
    m = dfs()
    dims, d = (33, 45, 80), 128
    n = 33 * 45 * 80
    heads = []
    for h in range(2):
        q, k, v = (bf16_round(x) for x in ora.gen_video_field(dims, d, 4.0, ora.derive_seed(1, [0, h])))
        heads.append((q, k, v))
    Q, K, V = (torch.from_numpy(np.stack([hd[i] for hd in heads], 1)).to(torch.bfloat16).cuda() for i in range(3))
    perm = m.hilbert3d_order(dims)
    qh, pq = m.ops.permute_to_hnd(Q, perm, 16)
    kh, pk = m.ops.permute_to_hnd(K, perm, 16)
    vh, _ = m.ops.permute_to_hnd(V, perm, 0)
    S = m.ops.score_pooled(pq, pk, n, m.ScoringParams(128, 16))
    lut = m.topk_lut(S, 0.1)
    assert lut.shape == (2, 929, 93)
    ptr = m.ops.lut_row_ptr(2, 929, 93)
    o = m.sparse_attention_csr(qh, kh, vh, ptr, lut.reshape(-1), 128)
    fwd = perm.forward.cpu().numpy().astype(np.uint32)
    rows = np.r_[0:256, 60000:60128, n - 144:n]
    for h in range(2):
        rq, rk, rv = (ora.apply_permutation(fwd, x) for x in heads[h])
        dense = np.zeros((929, 929), bool)
        dense[np.arange(929)[:, None], lut[h].cpu().numpy()] = True
        from oracle import dense_to_mask_bits

        bits = dense_to_mask_bits(dense)
        ref = np.zeros((n, d), np.float32)
        for lo, hi in [(0, 256), (60000, 60128), (n - 144, n)]:
            ref[lo:hi] = ora.block_sparse_attention(rq, rk, rv, bits, 929, 128, rows=(lo, hi))[lo:hi]
        got = o[h].float().cpu().numpy()[rows]
        err = np.abs(got - ref[rows]).max() / np.abs(ref[rows]).max()
        assert err <= 2e-2, (h, err)


@pytest.mark.parametrize("force_generic", [False, True])
def test_empty_csr_row_gives_zero_output(force_generic):
    """A caller-built CSR with an empty row (the BlockMask entry points refuse it, as
    attention.cpp:133-136 does) must not leak stale accumulators: the row is zero."""
    m = dfs()
    h, n, d = 2, 640, 128
    gen = torch.Generator().manual_seed(5)
    q, k, v = (torch.randn(h, n, d, generator=gen).to(torch.bfloat16).cuda() for _ in range(3))
    mq = n // 128
    counts = torch.tensor([[2, 0, 1, 3, 2], [0, 1, 1, 1, 5]], dtype=torch.int32)
    idx = []
    for hh in range(h):
        for u in range(mq):
            idx.append(torch.arange(int(counts[hh, u]), dtype=torch.int32))
    ptr = torch.zeros(h * mq + 1, dtype=torch.int32)
    ptr[1:] = torch.cumsum(counts.reshape(-1), 0)
    o = m.sparse_attention_csr(q, k, v, ptr.cuda(), torch.cat(idx).cuda(), 128, force_generic=force_generic)
    torch.cuda.synchronize()
    assert torch.isfinite(o.float()).all()
    assert (o[0, 128:256].float() == 0).all() and (o[1, 0:128].float() == 0).all()
    assert (o[0, 0:128].float().abs().sum() > 0)


def test_fuzz_tcgen05_vs_fp32_torch_reference():
    """Random geometries through K5 (tcgen05) and the SIMT kernel against a plain torch fp32
    softmax attention under the same block lists: N from 1 to 5000 (partial last blocks),
    1-3 heads, d in {64, 128}, K from 1 to M (dense lists included), HND and NHD inputs,
    optional gathered queries and scattered outputs."""
    m = dfs()
    rng = np.random.default_rng(2024)
    for trial in range(10):
        n = int(rng.integers(1, 5000))
        h = int(rng.integers(1, 4))
        d = int(rng.choice([64, 128]))
        mq = -(-n // 128)
        k = int(rng.integers(1, mq + 1))
        gen = torch.Generator().manual_seed(trial)
        q, kk, v = (torch.randn(h, n, d, generator=gen).to(torch.bfloat16).cuda() for _ in range(3))
        lut = random_lut(h, mq, mq, k, gen).cuda()
        ptr = m.ops.lut_row_ptr(h, mq, k)
        perm = torch.from_numpy(rng.permutation(n).astype(np.int32)).cuda()
        gather = bool(rng.integers(0, 2))
        qin = q
        if gather:  # queries arrive in raster rows [N, H, d]: q_raster[perm[i]] = q[:, i]
            qin = torch.empty(n, h, d, dtype=q.dtype, device=q.device)
            qin[perm.long()] = q.transpose(0, 1)
        o_fast = m.sparse_attention_csr(qin, kk, v, ptr, lut.reshape(-1), 128, layout=1, out_layout=1,
                                        in_rows=perm if gather else None)
        o_slow = m.sparse_attention_csr(qin, kk, v, ptr, lut.reshape(-1), 128, layout=1, out_layout=1,
                                        in_rows=perm if gather else None, force_generic=True)
        torch.cuda.synchronize()
        # torch fp32 reference
        qf, kf, vf = q.float(), kk.float(), v.float()
        ref = torch.empty(h, n, d, device="cuda")
        for hh in range(h):
            s = qf[hh] @ kf[hh].T / d ** 0.5
            allowed = torch.zeros(mq, mq, dtype=torch.bool, device="cuda")
            allowed[torch.arange(mq, device="cuda")[:, None], lut[hh].long()] = True
            keymask = allowed.repeat_interleave(128, 0)[:n].repeat_interleave(128, 1)[:, :n]
            s = s.masked_fill(~keymask, float("-inf"))
            ref[hh] = torch.softmax(s, -1) @ vf[hh]
        for name, o in (("tcgen05", o_fast), ("simt", o_slow)):
            err = float((o.float() - ref).abs().max() / ref.abs().max())
            assert err <= 2e-2, (trial, name, n, h, d, k, gather, err)


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("jump", [0.5, 6.0, 12.0, 40.0, 400.0])
def test_logit_jump_across_blocks(jump, d):
    """Online-softmax rescaling under large row-max jumps: key block 3 carries logits
    `jump` log2 units above block 0's (400 would overflow fp32 without the O/l rescale,
    0.5 and 6 stay under the lazy-rescale test — a half-row's block sum of p <= 2^12 —
    12 crosses it). Output must match a torch fp32 softmax, and a following ordinary call
    must be unaffected."""
    m = dfs()
    gen = torch.Generator().manual_seed(7)
    h, n = 2, 1024 + 40
    q = torch.full((h, n, d), 1.0) + 0.05 * torch.randn(h, n, d, generator=gen)
    kk = 0.05 * torch.randn(h, n, d, generator=gen)
    # logit_log2 = q.k / sqrt(d) * log2(e): choose block 3's key scale for the requested jump
    c = jump / (d / d ** 0.5 * 1.4426950408889634)
    kk[:, 3 * 128:4 * 128] += c
    v = torch.randn(h, n, d, generator=gen)
    q, kk, v = (x.to(torch.bfloat16).cuda() for x in (q, kk, v))
    mq = -(-n // 128)
    lut = torch.arange(mq, dtype=torch.int32).repeat(h, mq, 1).cuda()
    ptr = m.ops.lut_row_ptr(h, mq, mq)
    for _ in range(2):
        o = m.sparse_attention_csr(q, kk, v, ptr, lut.reshape(-1), 128, layout=1, out_layout=1)
        torch.cuda.synchronize()
        ref = torch.softmax(q.float() @ kk.float().transpose(1, 2) / d ** 0.5, -1) @ v.float()
        assert torch.isfinite(o.float()).all()
        assert rel(o.float(), ref) <= 2e-2, rel(o.float(), ref)
    # an ordinary call after the recovery pass
    q2, k2, v2 = (torch.randn(h, n, d, generator=gen).to(torch.bfloat16).cuda() for _ in range(3))
    o2 = m.sparse_attention_csr(q2, k2, v2, ptr, lut.reshape(-1), 128, layout=1, out_layout=1)
    ref2 = torch.softmax(q2.float() @ k2.float().transpose(1, 2) / d ** 0.5, -1) @ v2.float()
    assert rel(o2.float(), ref2) <= 2e-2


def test_output_only_16_byte_aligned():
    """The epilogue uses 32-byte stores when the output is 32-byte aligned and 16-byte
    stores otherwise: an output view offset by 16 bytes gives the same rows."""
    m = dfs()
    gen = torch.Generator().manual_seed(11)
    h, n, d = 2, 1000, 128
    q, kk, v = (torch.randn(h, n, d, generator=gen).to(torch.bfloat16).cuda() for _ in range(3))
    mq = -(-n // 128)
    lut = random_lut(h, mq, mq, 3, gen).cuda()
    ptr = m.ops.lut_row_ptr(h, mq, 3)
    flat = torch.zeros(n * h * d + 16, dtype=torch.bfloat16, device="cuda")
    out16 = flat[8:8 + n * h * d].view(n, h, d)
    assert out16.data_ptr() % 32 == 16
    o_al = m.sparse_attention_csr(q, kk, v, ptr, lut.reshape(-1), 128, out_layout=1)
    o_16 = m.sparse_attention_csr(q, kk, v, ptr, lut.reshape(-1), 128, out_layout=1, out=out16)
    torch.cuda.synchronize()
    assert o_al.data_ptr() % 32 == 0
    assert torch.equal(o_al.reshape(-1), o_16.reshape(-1))  # same NHD memory image


@pytest.mark.parametrize("nk", [77, 226, 512])
def test_text_cross_attention_shapes(nk):
    """Video queries attending to a short text sequence (Nk < one or a few key blocks,
    partial last block) through K5 with a full list, against a torch fp32 reference."""
    m = dfs()
    gen = torch.Generator().manual_seed(nk)
    h, nq, d = 3, 4096 + 64, 128
    q = torch.randn(nq, h, d, generator=gen).to(torch.bfloat16).cuda()
    k = torch.randn(nk, h, d, generator=gen).to(torch.bfloat16).cuda()
    v = torch.randn(nk, h, d, generator=gen).to(torch.bfloat16).cuda()
    o = m.full_attention_output(q, k, v)
    torch.cuda.synchronize()
    qf, kf, vf = (x.float().transpose(0, 1) for x in (q, k, v))
    ref = (torch.softmax(qf @ kf.transpose(1, 2) / d ** 0.5, -1) @ vf).transpose(0, 1)
    assert rel(o.float(), ref) <= 2e-2


def _random_csr(h, mq, mk, gen, kmax):
    """Ragged per-row key lists (1..kmax blocks, ascending) as a CSR over (head, query block)."""
    ptr, idx = [0], []
    for _ in range(h * mq):
        k = int(torch.randint(1, kmax + 1, (1,), generator=gen))
        sel = torch.randperm(mk, generator=gen)[:k].sort().values
        idx.append(sel)
        ptr.append(ptr[-1] + len(sel))
    return torch.tensor(ptr, dtype=torch.int32).cuda(), torch.cat(idx).to(torch.int32).cuda()


@pytest.mark.parametrize("d", [64, 128])
@pytest.mark.parametrize("n", [64, 256, 1000, 4096 + 33])
def test_sm100_block64_union_tiles(d, n):
    """B = 64 on tensor cores: a 128-row tile holds query blocks 2t and 2t+1 and walks the
    union of their (ragged, partly shared) key lists; each half attends only its own
    blocks (P = 0 elsewhere). Odd block counts leave a tile with one real query block;
    the partial last key block is masked (attention.cpp:146-152). vs the SIMT kernel."""
    m = dfs()
    gen = torch.Generator().manual_seed(n + d)
    h = 2
    q, kk, v = (torch.randn(h, n, d, generator=gen).to(torch.bfloat16).cuda() for _ in range(3))
    mb = -(-n // 64)
    ptr, idx = _random_csr(h, mb, mb, gen, kmax=min(mb, 6))
    o_fast = m.sparse_attention_csr(q, kk, v, ptr, idx, 64)
    o_ref = m.sparse_attention_csr(q, kk, v, ptr, idx, 64, force_generic=True)
    torch.cuda.synchronize()
    for hh in range(h):
        assert rel(o_fast[hh].float(), o_ref[hh].float()) <= 1e-2, hh
    # dense at B = 64 (full list, both halves own every block) and Nq != Nk
    qn = q.transpose(0, 1).contiguous()
    kn = torch.randn(n + 50, h, d, generator=gen).to(torch.bfloat16).cuda()
    vn = torch.randn(n + 50, h, d, generator=gen).to(torch.bfloat16).cuda()
    o = m.full_attention_output(qn, kn, vn, block=64)
    og = m.full_attention_output(qn, kn, vn, block=64, force_generic=True)
    assert rel(o.float(), og.float()) <= 1e-2


def test_bf16_unsupported_geometry_is_refused():
    """No silent SIMT fallback on the bf16 path: d = 96 or B = 32 raise
    UnsupportedGeometry unless the caller asks for the SIMT kernel."""
    m = dfs()
    for n, d, b in ((300, 96, 128), (300, 64, 32)):
        q = torch.randn(n, 2, d).to(torch.bfloat16).cuda()
        with pytest.raises(m._capi.UnsupportedGeometry):
            m.full_attention_output(q, q, q, block=b)
        m.full_attention_output(q, q, q, block=b, force_generic=True)  # explicit opt-in runs
