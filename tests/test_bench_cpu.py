"""bench.py host logic without a GPU: the workload table matches BASELINE.json's configs,
the headline metric name, and the executed-FLOP count of a block list."""
import json
import os

import pytest

torch = pytest.importorskip("torch")

import bench  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_workloads_match_baseline_configs():
    cfgs = json.load(open(os.path.join(ROOT, "BASELINE.json")))["configs"]
    text = " ".join(cfgs).replace("×", "x").replace(",", "")
    for key, (tokens, heads, d) in {"C": ("17550", 48, 64), "W4": ("32760", 40, 128), "HY": ("118800", 24, 128),
                                    "W7": ("75600", 40, 128)}.items():
        w = bench.WORKLOADS[key]
        f, hh, ww = w["dims"]
        assert str(f * hh * ww) == tokens and tokens in text, key
        assert (w["heads"], w["d"]) == (heads, d), key
        assert f"{heads} heads" in text and f"d={d}" in text


def test_headline_metric_is_baselines():
    base = json.load(open(os.path.join(ROOT, "BASELINE.json")))["metric"]
    m = bench.metric_for("HY")
    assert "HunyuanVideo" in base and "HunyuanVideo" in m and "90% sparsity" in m
    assert bench.metric_for("W7") != m  # other configs name themselves


def test_executed_flops_counts_real_tokens():
    # 2 heads, M = 3 blocks of 128 with a 40-token last block, every row keeps blocks {0, 2}
    n, block, d = 2 * 128 + 40, 128, 64
    lut = torch.tensor([[[0, 2]] * 3] * 2, dtype=torch.int32)
    rows = [128, 128, 40]
    cols = 128 + 40
    want = 4.0 * d * sum(r * cols for r in rows) * 2
    assert bench.executed_flops(lut, n, block, d) == pytest.approx(want)
