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
SUITES = ["test_curve", "test_attention", "test_mask_builder", "test_scheduler"]


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
