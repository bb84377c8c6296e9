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
    assert bench.metric_for("cfg2", 131072).startswith("decode tokens/s at 128K ctx")
    for w in ("cfg1", "cfg3", "cfg5"):
        assert bench.WORKLOADS[w]["desc"] in bench.metric_for(w, bench.WORKLOADS[w]["ctx"])
    # --ctx is reflected in the metric and the workload description
    assert bench.metric_for("cfg2", 32768).startswith("decode tokens/s at 32K ctx")
    assert "32K ctx" in bench.metric_for("cfg3", 32768)
    assert "64K ctx" in bench.metric_for("cfg3", 65536) and "32K" not in bench.metric_for("cfg3", 65536)


def test_config_identical_in_both_arms(bench, monkeypatch):
    # the reference arm and ours build `config` from the same function with
    # the same world size and per-GPU streams
    for argv, world in ((["bench.py"], 1), (["bench.py", "--gpus", "2"], 2),
                        (["bench.py", "--workload", "cfg3", "--gpus", "4"], 4)):
        monkeypatch.setattr(sys, "argv", argv)
        a = bench.parse()
        S = a.w["layers"] * a.w["kv_heads"] * a.w["batch"]
        c = bench.make_config(a, world, S // world)
        assert c["streams"] == S and c["streams_per_gpu"] * world == S
        assert c["ctx"] == a.w["ctx"]
        assert (c["parallelism"] == "single") == (world == 1)


def test_self_launch_builds_torchrun(bench, monkeypatch):
    # --gpus N outside torchrun re-launches N ranks under torch.distributed.run
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2", "--steps", "3"])
    monkeypatch.setenv("TTKV_SHARE_DEVICE", "1")
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    a = bench.parse()
    seen = {}

    def fake_call(cmd, env=None):
        seen["cmd"], seen["env"] = cmd, env
        return 0

    monkeypatch.setattr(bench.subprocess, "call", fake_call)
    with pytest.raises(SystemExit) as e:
        bench.self_launch(a)
    assert e.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:4] == ["-m", "torch.distributed.run", "--nnodes=1"]
    assert "--nproc-per-node=2" in cmd and "--master-addr=127.0.0.1" in cmd
    assert cmd[-3:] == ["--gpus", "2", "--steps", "3"][-3:]
    assert seen["env"]["NCCL_DEBUG"] == "INFO"


def test_self_launch_fails_without_devices(bench, monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "8"])
    monkeypatch.delenv("TTKV_SHARE_DEVICE", raising=False)
    a = bench.parse()
    with pytest.raises(SystemExit) as e:  # this container has no GPU
        bench.self_launch(a)
    assert e.value.code == 2


def test_world_size_must_match_gpus(bench, monkeypatch):
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "2"])
    monkeypatch.setenv("WORLD_SIZE", "4")
    with pytest.raises(SystemExit):
        bench.main()


def test_clock_summary_admissibility(bench):
    c = bench.Clocks(0)
    c.samples = [(1965.0, 1965.0, 0)] * 4 + [(1900.0, 1965.0, 0x4)]
    s = c.summary()
    assert s["samples"] == 5 and s["admissible"] and s["reasons"] == ["sw_power_cap"]
    assert s["sm_mhz"] == 1965.0 and s["sm_mhz_min"] == 1900.0
    c.samples = c.samples[:2]
    assert not c.summary()["admissible"]


def test_reference_line_ms_is_the_sample(bench, monkeypatch, capsys):
    # the reference arm prints what actually ran (sample ms/step, steps) and
    # the extrapolation factor in its own field
    import json
    import numpy as np
    monkeypatch.setattr(sys, "argv", ["bench.py", "--impl", "reference", "--steps", "4"])
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(bench, "ref_sample",
                        lambda ctx, n, G, engines=None, threads=None:
                        (np.full(n, 400.0), 1.0, 16, 16))
    bench.main()
    line = json.loads(capsys.readouterr().out.strip().splitlines()[-1])
    assert line["ms_per_step"] == 400.0 and line["steps"] == 4
    assert line["extrapolation"]["factor"] == 64.0
    assert line["value"] == pytest.approx(1000.0 / (64 * 400.0))
    assert line["config"] == bench.make_config(bench.parse(), 1, 256)
