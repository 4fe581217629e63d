"""CPU-side checks of the C ABI: the library loads, exports every declared
symbol, and its host-only logic (schedule, top-K count) matches the oracle.
No kernel is launched here (no GPU in the build container)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from oracle import ora

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_exports_every_declared_symbol():
    from paper_2605_23445_b200 import _capi

    header = open(os.path.join(ROOT, "include", "dfs_gpu.h")).read()
    declared = set(re.findall(r"^(?:int|const char\*)\s+(dfs_\w+)\(", header, re.M))
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(_capi.lib, name), name
    assert declared == set(_capi.EXPORTS), declared ^ set(_capi.EXPORTS)
    assert _capi.lib.dfs_abi_version() == 2


@pytest.mark.parametrize("case", [
    dict(total=50, warmup=0.25, budgets=(0.3, 0.2, 0.1), phase=0.25, interval=12),
    dict(total=23, warmup=0.2, budgets=(0.5, 0.25), phase=0.4, interval=3),
    dict(total=97, warmup=0.25, budgets=(0.3, 0.2, 0.1), phase=0.25, interval=7),
    dict(total=1, warmup=0.0, budgets=(0.1,), phase=1.0, interval=1),
    dict(total=50, warmup=1.0, budgets=(), phase=0.0, interval=12),
])
def test_schedule_matches_oracle(case):
    from paper_2605_23445_b200.ops import SparsitySchedule, ScheduleConfig

    s = SparsitySchedule(ScheduleConfig(case["total"], case["warmup"], case["budgets"], case["phase"],
                                        case["interval"]))
    b, u, ws, pl = ora.schedule(**case)
    assert s.warmup_steps() == ws and s.phase_length() == pl
    for t in range(case["total"]):
        got = s.budget_at(t)
        assert (got is None and b[t] < 0) or got == b[t]
        assert s.is_update_step(t) == bool(u[t])
    with pytest.raises(IndexError):
        s.budget_at(case["total"])
    with pytest.raises(IndexError):
        s.budget_at(-1)


def test_schedule_validation_errors():
    from paper_2605_23445_b200.ops import SparsitySchedule, ScheduleConfig

    for bad in [ScheduleConfig(total_steps=0), ScheduleConfig(phase_budgets=(0.3, 1.5)),
                ScheduleConfig(warmup_fraction=0.5, phase_fraction=0.25),
                ScheduleConfig(warmup_fraction=0.5, phase_budgets=())]:
        with pytest.raises(ValueError):
            SparsitySchedule(bad)


def test_topk_count_matches_oracle():
    from paper_2605_23445_b200 import topk_count

    rng = np.random.default_rng(3)
    for _ in range(200):
        m = int(rng.integers(1, 3000))
        g = float(rng.uniform(1e-4, 1.0))
        assert topk_count(g, m) == ora.topk_count(g, m)
    assert topk_count(0.5, 5) == 3 and topk_count(0.01, 10) == 1 and topk_count(0.1, 929) == 93
    for bad in (0.0, -0.1, 1.5):
        with pytest.raises(ValueError):
            topk_count(bad, 4)
