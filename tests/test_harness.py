"""Harness on the B200 engine (paper_2604_19769_b200/harness.py) vs the
reference harness (harness.cpp).

CPU: baseline emulation rules and the aggregation/report format.
GPU: the reference's own ablation and criterion-3 numbers, reproduced exactly
by the GPU engine's accounting (acceptance.cpp:172-195 and 430-465).
"""
import os

import numpy as np

import pytest

from paper_2604_19769_b200 import harness as H
from paper_2604_19769_b200.engine import SelectionPolicy, TierConfig


def test_effective_config_rules():
    # harness.cpp:56-86 and 22-24
    base = TierConfig(d_k=64, d_v=64)
    pol = SelectionPolicy(None, 0.45)
    t, p, serial = H.effective(base, pol, "ttkv")
    assert t.hbm_budget_bytes == 1024 * 128 * 2 and p.fetch_fraction == 0.45 and not serial
    t, p, serial = H.effective(base, pol, "fp16_full_fetch")
    assert (t.key_bits, t.value_bits, p.fetch_fraction, serial) == (16, 16, 1.0, True)
    t, p, serial = H.effective(base, pol, "uniform_quant_8_8")
    assert (t.key_bits, t.value_bits, serial) == (8, 8, False)
    t, p, serial = H.effective(base, pol, "single_tier")
    assert t.hbm_budget_bytes == t.block_bytes_full_precision() and p.fetch_fraction == 1.0
    t, p, serial = H.effective(base, pol, "no_pipeline")
    assert serial and (t.key_bits, t.value_bits) == (8, 4)
    with pytest.raises(ValueError):
        H.effective(base, pol, "nope")


def test_aggregate_nearest_rank_and_warmup():
    # aggregate_run (sim.cpp:152-184): 5 warm-up steps dropped at >= 25 steps
    r = H.RunRecord("ttkv", H.WorkloadSpec(), TierConfig(), SelectionPolicy())
    r.latency_ms = [100.0] * 5 + [float(i) for i in range(1, 21)]
    r.step_bytes = [10.0] * 25
    r.baseline_bytes = [50.0] * 25
    r.pcie_bytes = [0] * 25
    s = H.aggregate(r)
    assert s["p95_latency_ms"] == 19.0  # ceil(0.95 * 20) = 19th of 1..20
    assert s["traffic_reduction"] == 5.0
    r.step_bytes = [0.0] * 25
    assert H.aggregate(r)["traffic_reduction"] == float("inf")


def test_report_format(tmp_path):
    r = H.RunRecord("ttkv", H.WorkloadSpec(), TierConfig(), SelectionPolicy())
    r.latency_ms, r.step_bytes, r.baseline_bytes, r.pcie_bytes = [1.0], [2.0], [3.0], [4]
    r.blocks_scored, r.blocks_fetched, r.evictions, r.oracle_errors = [5], [6], [True], [0.5]
    r.summary = H.aggregate(r)
    csv = H.write_report([r])
    assert csv.splitlines()[0] == ",".join(H.REPORT_COLUMNS)
    H.emit_report([r], str(tmp_path))
    assert (tmp_path / "report.csv").exists() and (tmp_path / "steps-000.csv").exists()
    with pytest.raises(ValueError):
        H.write_report([])


@pytest.mark.gpu
def test_ablation_traffic_matches_reference(gpu):
    """acceptance.cpp:430-465 defaults (d=64, block 128, 8/4, 0.45, 4K ctx,
    seed 42, 32 steps): H->G bytes per method from the unmodified reference."""
    recs = H.run_ablation(TierConfig(d_k=64, d_v=64), SelectionPolicy(None, 0.45),
                          H.WorkloadSpec(context_length=4096, decode_steps=32, seed=42),
                          oracle=False)
    got = {r.method: r.summary["total_h2g_bytes"] for r in recs}
    assert got == {"fp16_full_fetch": 26181632.0, "single_tier": 13094400.0,
                   "uniform_quant_8_8": 6471168.0, "no_pipeline": 4902400.0,
                   "ttkv": 4902400.0}
    for r in recs:
        assert all(l > 0 for l in r.latency_ms)


@pytest.mark.gpu
def test_criterion3_traffic_reduction_on_gpu(gpu):
    # acceptance.cpp:172-195: 5.638997722095672x at 16K, d=128, 1024-token fast tier
    tier = TierConfig(hbm_budget_bytes=1024 * 256 * 2, d_k=128, d_v=128)
    rec = H.run_benchmark(tier, SelectionPolicy(None, 0.45),
                          H.WorkloadSpec(context_length=16384, decode_steps=8, d_k=128, d_v=128,
                                         seed=3))
    assert rec.summary["total_h2g_bytes"] == 11238400.0
    assert abs(rec.summary["traffic_reduction"] - 5.638997722095672) < 1e-12
    # with 8/4 + 45 % the engine sits ~0.98 L2-relative from dense
    assert all(0.5 < e < 1.2 for e in rec.oracle_errors)


@pytest.mark.gpu
def test_needle_recall_through_harness(gpu):
    tier = TierConfig(d_k=64, d_v=1, hbm_budget_bytes=1024 * 65 * 2)
    rec = H.run_benchmark(tier, SelectionPolicy(None, 0.45),
                          H.WorkloadSpec(kind="needle", context_length=4096, decode_steps=4,
                                         d_k=64, d_v=1, seed=40000), oracle=False)
    assert rec.needle_hits == 4  # seed 40000 is a hit at B=128 (tests/golden/needle.json)


@pytest.mark.gpu
def test_emit_report_on_gpu(gpu, tmp_path):
    recs = H.run_sweep(TierConfig(d_k=32, d_v=32, block_size=64, hbm_budget_bytes=256 * 64 * 2),
                       SelectionPolicy(None, 0.45),
                       H.WorkloadSpec(context_length=1024, decode_steps=6, d_k=32, d_v=32,
                                      seed=77), context_lengths=(768, 1024),
                       fetch_fractions=(0.3, 0.45))
    H.emit_report(recs, str(tmp_path), "json")
    assert len(os.listdir(tmp_path)) == 5


@pytest.mark.gpu
def test_measured_timelines_on_gpu(gpu):
    # write_run_timelines (harness.cpp:291-300) from measured kernel events
    spec = H.WorkloadSpec(context_length=6000, decode_steps=4, d_k=64, d_v=64, seed=5)
    rec = H.run_benchmark(TierConfig(d_k=64, d_v=64, block_size=128,
                                     hbm_budget_bytes=1024 * 128 * 2),
                          SelectionPolicy(None, 0.45), spec)
    assert len(rec.timelines) == 4
    for tl, lat in zip(rec.timelines, rec.latency_ms):
        names = [n for n, _, _ in tl]
        # score + select run as one fused kernel ("select") up to 2048 blocks
        assert {"append", "select", "fast", "slow", "combine"} <= set(names)
        for _, a, b in tl:
            assert -1e-3 <= a <= b <= lat + 1e-3
    tsv = H.write_run_timelines(rec).splitlines()
    assert len(tsv) == sum(len(t) for t in rec.timelines)
    f = tsv[0].split("\t")
    assert f[0] == "0" and f[1] in ("compute", "transfer") and len(f) == 5
    assert any(line.split("\t")[1:3] == ["transfer", "slow"] for line in tsv)


def test_dropin_workload_generator_matches_reference():
    # libttkv.so's generate_workload (C entry in include/ttkv_dropin_c.h) is the
    # reference generator (workload.cpp:42-95), pinned against the oracle port
    import numpy as np
    import _oracle as O
    got = H.generate_workload(H.WorkloadSpec(context_length=300, decode_steps=5, d_k=16, d_v=16,
                                             seed=13))
    want = O.generate_workload(300, 5, 16, 16, 13)
    assert all(np.array_equal(a, b) for a, b in zip(got, want))
    got = H.generate_workload(H.WorkloadSpec(kind="needle", context_length=1024, decode_steps=2,
                                             d_k=64, d_v=1, seed=40001))
    want = O.generate_workload(1024, 2, 64, 1, 40001, needle=True)
    assert all(np.array_equal(a, b) for a, b in zip(got, want))


# ---------------------------------------------------------------------------
# the timing model restated in harness.py == the reference's sim.cpp (CPU)
# ---------------------------------------------------------------------------
def _ref_sim(pipelined, compute, transfers, bw, lat, rate):
    import ctypes as C
    import _oracle as O
    lib = O.ref()
    f = lib.ref_simulate
    f.restype = C.c_int
    ca = np.asarray(compute, np.float64)
    ta = np.asarray([t for _, t in transfers] or [0.0], np.float64)
    to = np.asarray([i for i, _ in transfers] or [0], np.uint64)
    out = [C.c_double() for _ in range(5)]
    rc = f(C.c_int(int(pipelined)), C.c_uint64(len(compute)), ca.ctypes.data_as(C.c_void_p),
           C.c_uint64(len(transfers)), ta.ctypes.data_as(C.c_void_p),
           to.ctypes.data_as(C.c_void_p), C.c_double(bw), C.c_double(lat), C.c_double(rate),
           *[C.byref(o) for o in out])
    assert rc == 0
    return [o.value for o in out]


@pytest.mark.skipif(not __import__("_oracle").ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("seed", range(6))
def test_sim_matches_reference(seed):
    from paper_2604_19769_b200 import harness as H
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 40))
    compute = list(rng.uniform(1e3, 1e6, n))
    idx = sorted(rng.choice(np.arange(1, n), size=min(n - 1, int(rng.integers(0, n))),
                            replace=False).tolist()) if n > 1 else []
    rng.shuffle(idx)  # transfer order = schedule order of the reference's report
    transfers = [(int(i), float(rng.uniform(1e3, 1e5))) for i in idx]
    bw, lat, rate = float(rng.uniform(1e9, 6e10)), float(rng.choice([0.0, 2e-6])), 1e9
    for pipelined in (False, True):
        fn = H.simulate_pipelined if pipelined else H.simulate_serial
        tl = fn(compute, transfers, H.LinkModel(bw, lat), rate)
        ref = _ref_sim(pipelined, compute, transfers, bw, lat, rate)
        got = [tl.total_latency, tl.idle_fraction, tl.mean_transfer_stall, tl.total_compute,
               tl.total_transfer]
        assert np.allclose(got, ref, rtol=1e-12, atol=0), (pipelined, got, ref)


# ---------------------------------------------------------------------------
# RunConfig files (harness.cpp:324-413) vs the reference's own parser (CPU)
# ---------------------------------------------------------------------------
CONFIG_CASES = [
    "",
    "# only a comment\n\n   \n",
    "seed = 7\ncontext_length=16384\ndecode_steps = 8 # trailing comment\nd_k=128\nd_v = 96\n",
    "workload = planted_needle\nneedle_block_position = 3\nneedle_alignment_strength = 2.5\n",
    "hbm_budget_bytes = 524288\nblock_size = 64\nkey_bits = 6\nvalue_bits = 3\n"
    "bytes_full_precision = 4\nfetch_fraction = 0.3\ntop_k_blocks = 12\n",
    "hbm_bandwidth = 8e12\npcie_bandwidth=5.5e10\ntransfer_latency = 2e-6\ncompute_rate = 1e13\n",
    "baseline = no_pipeline\nformat = json\nout_dir = /tmp/x y\nliteral_merge = true\r\n",
    "seed = 12abc\nkey_bits = 4294967304\n",            # prefix parse, unsigned wrap
    "seed = -1\n",                                       # stoull negation wraps
    "fetch_fraction = .5e1x\n",
    "seed = abc\n",                                      # bad value
    "seed = 99999999999999999999999\n",                  # out of range
    "compute_rate = 1e999\n",                            # out of range
    "workload = uniform\n",                              # unknown kind
    "baseline = fastest\n",                              # unknown baseline
    "format = xml\n",                                    # unknown format
    "colour = blue\n",                                   # unknown key
    "seed 7\n",                                          # expected key = value
    "seed = 1\nseed = 2\n",                              # last wins
]


def _ref_load(path):
    import ctypes as C
    import _oracle as O
    f = O.ref().ref_load_config
    f.restype = C.c_int
    u64 = np.zeros(9, np.uint64)
    u32 = np.zeros(7, np.uint32)
    f64 = np.zeros(7, np.float64)
    tk = C.c_uint64()
    out = C.create_string_buffer(256)
    rc = f(str(path).encode(), u64.ctypes.data_as(C.c_void_p), u32.ctypes.data_as(C.c_void_p),
           f64.ctypes.data_as(C.c_void_p), C.byref(tk), out, C.c_uint64(256))
    return rc, O.ref().ref_last_error().decode(), u64, u32, f64, tk.value, out.value.decode()


@pytest.mark.skipif(not __import__("_oracle").ref_available(), reason="oracle/_ref not built")
@pytest.mark.parametrize("i", range(len(CONFIG_CASES)))
def test_config_file_matches_reference(tmp_path, i):
    from paper_2604_19769_b200.engine import ConfigError as CE
    path = tmp_path / "run.cfg"
    path.write_bytes(CONFIG_CASES[i].encode())
    rc, msg, u64, u32, f64, top_k, out_dir = _ref_load(path)
    if rc != 0:
        assert rc == 1, msg
        with pytest.raises(CE) as e:
            H.load_run_config(path)
        assert str(e.value) == msg
        return
    cfg, spec = H.load_run_config(path)
    t = cfg.tier
    assert [spec.seed, spec.context_length, spec.decode_steps, spec.d_k, spec.d_v,
            spec.needle_block_position, t.hbm_budget_bytes, t.block_size,
            t.bytes_full_precision] == [int(x) for x in u64]
    assert [int(spec.kind == "needle"), t.key_bits, t.value_bits,
            int(cfg.policy.top_k is not None), H.BASELINES.index(cfg.baseline),
            ["csv", "json"].index(cfg.format), int(cfg.literal_merge)] == [int(x) for x in u32]
    assert [spec.needle_alignment_strength, t.fetch_fraction, cfg.policy.fetch_fraction,
            t.hbm_bandwidth, t.pcie_bandwidth, t.transfer_latency, t.compute_rate] == list(f64)
    assert (cfg.policy.top_k or 0) == top_k and cfg.out_dir == out_dir


def test_config_file_missing_is_io_error(tmp_path):
    from paper_2604_19769_b200.engine import IoError
    with pytest.raises(IoError, match="cannot open config file"):
        H.load_run_config(tmp_path / "nope.cfg")
