"""Host-side logic of bench.py (CPU): argument defaults, the cfg5 growth
integral, the CPU-baseline extrapolation and the driver-facing JSON keys."""
import importlib
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def bench():
    sys.path.insert(0, ROOT)
    return importlib.import_module("bench")


def test_defaults_are_the_driver_contract(bench, monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py"])
    a = bench.parse()
    assert (a.gpus, a.steps, a.warmup, a.impl, a.workload) == (1, 10, 3, "ours", "cfg2")
    assert a.w["ctx"] == 131072 and a.w["layers"] * a.w["kv_heads"] == 256 and a.w["G"] == 4
    monkeypatch.setattr(sys, "argv", ["bench.py", "--workload", "cfg5"])
    assert not bench.parse().steps_given  # cfg5 then times one eviction period per point


def test_growth_integral(bench):
    # linear ms/step(ctx): the sustained rate is the mean of the end points
    curve = [{"ctx_start": c, "ms_per_step": 100.0 + (c - 131072) / 1000.0}
             for c in bench.GROWTH_POINTS]
    ms = bench.growth_ms_per_step(curve)
    assert ms == pytest.approx((curve[0]["ms_per_step"] + curve[-1]["ms_per_step"]) / 2)
    assert bench.growth_ms_per_step(curve[:1]) == curve[0]["ms_per_step"]


def test_cpu_baseline_extrapolation(bench):
    # 16 of 1024 engines in 450 ms -> 1024 engines take 64 x 450 ms per token
    assert bench.cpu_throughput(450.0, 16, 1024, 1) == pytest.approx(1000.0 / (64 * 450.0))
    assert bench.scale_note(32, 32) == "all engines, not extrapolated"
    assert "x64" in bench.scale_note(16, 1024)


def test_metric_names(bench):
    assert bench.metric_for("cfg2").startswith("decode tokens/s at 128K ctx")
    for w in ("cfg1", "cfg3", "cfg5"):
        assert bench.WORKLOADS[w]["desc"] in bench.metric_for(w)
