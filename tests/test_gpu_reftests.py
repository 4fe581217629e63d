"""The reference's own hot-path unit suites and acceptance criteria, unmodified,
relinked against the B200 drop-in library.

oracle/Makefile `reftests` compiles /root/reference/proj/tests/test_{curve,
attention,mask_builder,scheduler}.cpp and acceptance_main.cpp with our
include/dfs/*.hpp first on the include path, so every dfs:: hot-path call in
them (hilbert3d_order, apply_permutation, build_mask, topk_select,
block_sparse_attention, full_attention, run_step, run_trajectory, ...) resolves
to paper_2605_23445_b200/libdfs_b200.so and runs on the GPU; their off-path
helpers (io, rng, metrics, theory, synthetic, config, commands) are the
reference's own sources. The binaries are built in the container that has
/root/reference and travel to the GPU box prebuilt (oracle/_ref is git-ignored,
not gpurun-ignored); nothing here reads /root/reference at run time.
"""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "reftests")
SUITES = ["test_curve", "test_attention", "test_mask_builder", "test_scheduler", "test_cli"]


def _run(name, timeout=600):
    exe = os.path.join(BIN, name)
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C oracle reftests needs /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=timeout, cwd=BIN)
    return r


@pytest.mark.parametrize("suite", SUITES)
def test_reference_unit_suite_passes_on_gpu_library(suite):
    r = _run(suite)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-4000:])
    assert "0 failed" in r.stdout, r.stdout


def test_reference_acceptance_criteria_pass_on_gpu_library():
    r = _run("acceptance", timeout=1200)
    assert r.returncode == 0, (r.stdout[-4000:], r.stderr[-4000:])


RUN_CONFIGS = {
    # test_cli.cpp:36-52 small_run_config: 2 layers, updates at sparse steps 1, 3, 5
    "small": {"seed": 3, "total_steps": 6, "warmup_fraction": 0.2, "phase_budgets": [0.5, 0.25],
              "phase_fraction": 0.4, "update_interval": 2, "ordering": "hilbert3d", "block_size": 16,
              "sub_block_size": 4, "dims": [4, 4, 4], "head_dim": 8, "layers": 2, "heads": 1,
              "trajectory": {"smoothness": 2, "noise_start": 1.0, "noise_end": 0.0}},
    # the reference defaults' schedule (T = 50, warmup 25 %, budgets 0.3/0.2/0.1, Delta = 12) on a
    # 16^3 lattice with B = 64, B_s = 16, 2 layers x 2 heads, recall recorded (N = 4096 <= cap)
    "schedule50": {"seed": 11, "total_steps": 50, "warmup_fraction": 0.25, "phase_budgets": [0.3, 0.2, 0.1],
                   "phase_fraction": 0.25, "update_interval": 12, "ordering": "hilbert3d", "block_size": 64,
                   "sub_block_size": 16, "dims": [16, 16, 16], "head_dim": 32, "layers": 2, "heads": 2,
                   "trajectory": {"smoothness": 3, "noise_start": 1.5, "noise_end": 0.0}},
}


@pytest.mark.parametrize("name", sorted(RUN_CONFIGS))
def test_cmd_run_outputs_byte_identical_to_reference(name, tmp_path):
    """cmd_run (commands.cpp:221-319) end to end: the reference CLI code driving the
    B200 library writes the same report.csv (step, layer, head, budget, sparsity,
    recall at %.9g, mask_updated) and the same masks/*.dfsm files, byte for byte, as
    the same code driving the reference's own CPU library."""
    import json

    cfg = tmp_path / "run.json"
    cfg.write_text(json.dumps(RUN_CONFIGS[name]))
    outs = {}
    for tag in ("cmd_ref", "cmd_gpu"):
        exe = os.path.join(BIN, tag)
        if not os.path.exists(exe):
            pytest.skip(f"{exe} not built (make -C oracle reftests needs /root/reference)")
        out = tmp_path / tag
        r = subprocess.run([exe, "run", str(cfg), str(out), "2"], capture_output=True, text=True, timeout=1200)
        assert r.returncode == 0, (tag, r.stdout[-2000:], r.stderr[-2000:])
        outs[tag] = out
    ref, gpu = outs["cmd_ref"], outs["cmd_gpu"]
    assert (ref / "report.csv").read_bytes() == (gpu / "report.csv").read_bytes()
    ref_masks = sorted(p.name for p in (ref / "masks").iterdir())
    assert ref_masks and ref_masks == sorted(p.name for p in (gpu / "masks").iterdir())
    for fname in ref_masks:
        assert (ref / "masks" / fname).read_bytes() == (gpu / "masks" / fname).read_bytes(), fname


def test_cmd_gpu_runs_the_north_star_shape(tmp_path):
    """The reference's own cmd_run (commands.cpp:221-319) driving the drop-in library at
    the HunyuanVideo-720p lattice (118,800 tokens, d = 128, B = 128, B_s = 16, gamma = 0.1)
    — past the 4096-row cap where the reference's block_scores throws: run_trajectory
    batches each layer's heads into one device step (fp32 pooling + the fp32-accurate
    tcgen05 scorer, K5 tcgen05 attention). The DFSM masks it writes must agree with the C
    oracle's masks on the same fp32 inputs on >= 99.5 % of bits; the
    report carries the streamed recall (recorded past the cap)."""
    import json

    import numpy as np

    from oracle import mask_bits_to_dense, ora

    exe = os.path.join(BIN, "cmd_gpu")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built")
    dims, d, heads = [33, 45, 80], 128, 2
    cfg = {"seed": 5, "total_steps": 2, "warmup_fraction": 0.5, "phase_budgets": [0.1], "phase_fraction": 0.5,
           "update_interval": 1, "ordering": "hilbert3d", "block_size": 128, "sub_block_size": 16, "dims": dims,
           "head_dim": d, "layers": 1, "heads": heads,
           "trajectory": {"smoothness": 4, "noise_start": 0.5, "noise_end": 0.0}}
    (tmp_path / "run.json").write_text(json.dumps(cfg))
    out = tmp_path / "out"
    r = subprocess.run([exe, "run", str(tmp_path / "run.json"), str(out), str(os.cpu_count() or 4)],
                       capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, (r.stdout[-2000:], r.stderr[-2000:])
    rows = (out / "report.csv").read_text().strip().splitlines()
    assert len(rows) == 1 + 2 * heads
    n = dims[0] * dims[1] * dims[2]
    m = -(-n // 128)
    k = ora.topk_count(0.1, m)
    fwd = ora.hilbert3d_order(dims)
    for head in range(heads):
        raw = (out / "masks" / f"mask_step001_layer00_head{head:02d}.dfsm").read_bytes()
        assert raw[:4] == b"DFSM" and int.from_bytes(raw[8:12], "little") == m
        got = mask_bits_to_dense(np.frombuffer(raw[16:], np.uint8), m)
        assert (got.sum(1) == k).all()
        seed = ora.derive_seed(5, [head])
        q, kk, _ = ora.trajectory_at(dims, d, 4.0, seed, 2, 0.5, 0.0, 1)
        want = mask_bits_to_dense(ora.build_mask(ora.apply_permutation(fwd, q), ora.apply_permutation(fwd, kk),
                                                 128, 16, 0.1), m)
        assert (got == want).mean() >= 0.995, head
