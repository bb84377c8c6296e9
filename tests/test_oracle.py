"""The CPU oracle (oracle/ttkv_oracle.c) pinned against the reference's own
golden vectors and -- where oracle/_ref was built -- the unmodified reference.

Golden vectors (reference test files under /root/reference/proj/tests):
  test_quantizer.cpp:36-152, test_relevance.cpp:8-42, test_tier_store.cpp:30-46,
  test_engine.cpp:95-110, acceptance.cpp:172-195 (criterion 3) and 376-426
  (criterion 7), plus tests/golden/*.json generated from oracle/_ref by
  tests/golden/make_golden.py.
"""
import json
import os

import numpy as np
import pytest

import _oracle as O

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


# ---- quantizer golden vectors (test_quantizer.cpp) ---------------------------
def test_4bit_packing_golden():
    params, packed = O.quantize_tensor(np.array([[0.], [5.], [10.], [15.]]), 4)
    assert list(packed) == [0x50, 0xFA]
    assert params[0] == 1.0 and params[1] == 0.0
    back = O.dequantize_tensor(packed, 4, 1, 4, params)
    assert np.array_equal(back.ravel(), [0, 5, 10, 15])


def test_2bit_packing_golden():
    params, packed = O.quantize_tensor(np.array([[1.], [2.], [3.], [0.], [3.]]), 2)
    assert list(packed) == [0x39, 0x03]


def test_constant_channels_exact():
    k = np.tile(np.array([-4.25, 0.0, 1e-20], np.float32), (16, 1))
    params, packed = O.quantize_tensor(k, 8)
    assert np.array_equal(O.dequantize_tensor(packed, 16, 3, 8, params), k)


def test_error_bound_random_blocks():
    # test_quantizer.cpp:83-110
    rng = np.random.default_rng(11)
    for trial in range(200):
        bits = 4 if trial % 2 else 8
        x = rng.uniform(-3, 3, (24, 6)).astype(np.float32)
        params, packed = O.quantize_tensor(x, bits)
        back = O.dequantize_tensor(packed, 24, 6, bits, params)
        lo, hi = x.min(0).astype(np.float64), x.max(0).astype(np.float64)
        levels = (1 << bits) - 1
        bound = (hi - lo) / (2 * levels) + 4 * (hi - lo) * 1.19209290e-07
        assert (np.abs(back.astype(np.float64) - x) <= bound).all()


def test_passthrough_16bit_lossless():
    x = np.random.default_rng(3).uniform(-10, 10, (32, 8)).astype(np.float32)
    params, packed = O.quantize_tensor(x, 16)
    assert packed.size == 32 * 8 * 4
    assert np.array_equal(O.dequantize_tensor(packed, 32, 8, 16, params), x)


def test_modeled_block_bytes():
    L = O.oracle()
    assert L.tko_modeled_block_bytes(128, 128, 128, 8, 4) == 25600
    assert L.tko_modeled_block_bytes(128, 128, 128, 16, 16) == 65536
    assert L.tko_modeled_block_bytes(128, 128, 128, 8, 8) == 33792
    assert L.tko_modeled_block_bytes(128, 128, 128, 4, 4) == 17408


def test_centroid_prequant_mean():
    k = np.array([[1, 0], [2, 4], [3, 0], [6, 4]], np.float32)
    out = np.zeros(2, np.float32)
    O.oracle().tko_centroid(k.reshape(-1), 4, 2, out)
    assert out[0] == 3.0 and out[1] == 2.0


# ---- relevance golden vectors (test_relevance.cpp) ----------------------------
def test_policy_resolution():
    r = O.oracle().tko_resolve
    assert r(0, 0, 0.45, 10) == 5 and r(0, 0, 0.45, 1) == 1 and r(0, 0, 0.45, 0) == 0
    assert r(0, 0, 1.0, 7) == 7
    assert r(1, 5, 0.45, 3) == 3 and r(1, 5, 0.45, 20) == 5
    assert r(0, 0, 0.0, 5) == 2 ** 64 - 1  # ConfigError


def test_score_block():
    q = np.array([1, 2, -1], np.float32)
    c = np.array([0.5, 0.25, 4.0], np.float32)
    assert O.oracle().tko_score_block(q, c, 3) == 0.5 + 0.5 - 4.0


def test_top_k_tie_break():
    scores = np.array([1.0, 2.0, 2.0, 0.5, -1.0])
    out = np.zeros(5, np.uint64)
    O.oracle().tko_select_top_k(scores, None, 5, 2, out)
    assert list(out[:2]) == [2, 1]
    O.oracle().tko_select_top_k(scores, None, 5, 5, out)
    assert list(out) == [2, 1, 0, 3, 4]


# ---- tier store (test_tier_store.cpp:30-46, test_engine.cpp:95-110) ----------
def test_fast_capacity():
    fc = O.oracle().tko_fast_capacity
    assert fc(1048576, 256, 2, 128) == 2048
    assert fc(1048575, 256, 2, 128) == 1920
    assert fc(128 * 256 * 2 - 1, 256, 2, 128) == 0


def test_evictions_settle_fast_97():
    pk, pv, dk, dv, dq = O.generate_workload(160, 6, 16, 16, 13)
    e = O.OracleEngine(16, 16, 32, 128)
    e.prefill(pk, pv)
    assert e.fast_tokens() == 128
    r = e.decode_step(dq[0], dk[0], dv[0])
    assert r["eviction_occurred"] and e.fast_tokens() == 97


def test_lossless_fetch_all_equals_dense():
    # test_engine.cpp:35-48 (fp64 engine; < 1e-12)
    pk, pv, dk, dv, dq = O.generate_workload(512, 6, 16, 16, 13)
    e = O.OracleEngine(16, 16, 32, 128, 16, 16, None, 1.0)
    e.prefill(pk, pv)
    hk, hv = list(pk), list(pv)
    for t in range(6):
        r = e.decode_step(dq[t], dk[t], dv[t])
        hk.append(dk[t]); hv.append(dv[t])
        dense = np.zeros(16)
        O.oracle().tko_dense_attention(dq[t], 16, np.ascontiguousarray(hk).reshape(-1),
                                       np.ascontiguousarray(hv).reshape(-1), len(hk), 16, dense)
        assert O.oracle().tko_relative_error(r["output"][0], dense, 16) < 1e-12


def test_quantized_close_to_dense():
    # test_engine.cpp:50-62 (< 0.2)
    pk, pv, dk, dv, dq = O.generate_workload(512, 6, 16, 16, 13)
    e = O.OracleEngine(16, 16, 32, 128, 8, 4, None, 1.0)
    e.prefill(pk, pv)
    hk, hv = list(pk), list(pv)
    for t in range(6):
        r = e.decode_step(dq[t], dk[t], dv[t])
        hk.append(dk[t]); hv.append(dv[t])
        dense = np.zeros(16)
        O.oracle().tko_dense_attention(dq[t], 16, np.ascontiguousarray(hk).reshape(-1),
                                       np.ascontiguousarray(hv).reshape(-1), len(hk), 16, dense)
        assert O.oracle().tko_relative_error(r["output"][0], dense, 16) < 0.2


def test_step_report_accounting():
    # test_engine.cpp:64-93
    pk, pv, dk, dv, dq = O.generate_workload(512, 1, 16, 16, 13)
    e = O.OracleEngine(16, 16, 32, 128, 8, 4, None, 0.45)
    e.prefill(pk, pv)
    n = e.slow_blocks()
    r = e.decode_step(dq[0], dk[0], dv[0])
    k = O.oracle().tko_resolve(0, 0, 0.45, n)
    assert r["blocks_scored"] == n and len(r["fetched"][0]) == k
    assert r["bytes_transferred"] == k * O.oracle().tko_modeled_block_bytes(32, 16, 16, 8, 4)


# ---- committed golden fixtures (from the unmodified reference) ----------------
def _golden(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def test_golden_criterion3_fingerprint():
    """acceptance.cpp:172-195 operating point: seed 3, 16K ctx, fast tier 1024,
    d=128, K8/V4, 0.45, 8 steps.  The fetched lists and the H->G total were
    produced by oracle/_ref (tests/golden/make_golden.py)."""
    g = _golden("criterion3.json")
    pk, pv, dk, dv, dq = O.generate_workload(16384, 8, 128, 128, 3)
    e = O.OracleEngine(128, 128, 128, 1024)
    e.prefill(pk, pv)
    total = 0.0
    for t in range(8):
        r = e.decode_step(dq[t], dk[t], dv[t])
        assert [int(x) for x in r["fetched"][0]] == g["fetched"][t]
        assert np.allclose(r["output"][0], g["outputs"][t], rtol=0, atol=1e-15)
        total += r["bytes_transferred"]
    assert total == g["total_h2g_bytes"] == 11238400
    assert g["fetched"][0][:5] == [42, 51, 13, 118, 55]


def test_golden_serialized_blocks():
    g = _golden("blocks_small.json")
    pk, pv, *_ = O.generate_workload(g["ctx"], 1, g["d"], g["d"], g["seed"])
    e = O.OracleEngine(g["d"], g["d"], g["B"], g["l_fast"], g["kb"], g["vb"])
    e.prefill(pk, pv)
    assert e.slow_blocks() == len(g["blocks_hex"])
    for i, hx in enumerate(g["blocks_hex"]):
        assert e.serialize_block(i).hex() == hx


def test_golden_needle_recall_subset():
    """Criterion 7 (acceptance.cpp:376-426) on the first 100 seeds: the
    per-seed hit/miss fingerprint of the reference at B=128 and B=256."""
    g = _golden("needle.json")
    for B in (128, 256):
        hits = []
        for t in range(100):
            pk, pv, *_ = O.generate_workload(4096, 0, 64, 1, 40000 + t, needle=True)
            e = O.OracleEngine(64, 1, B, 1024 // B * B if B <= 1024 else B)
            e.prefill(pk, pv)
            n = e.slow_blocks()
            scores = np.array([O.oracle().tko_score_block(np.full(64, 1 / 8, np.float32),
                                                          e.centroid(i), 64) for i in range(n)])
            k = O.oracle().tko_resolve(0, 0, 0.45, n)
            sel = np.zeros(max(k, 1), np.uint64)
            O.oracle().tko_select_top_k(scores, None, n, k, sel)
            needle_block = 256 // B
            hits.append(int(needle_block in sel[:k]))
        assert hits == g[str(B)]


# ---- the unmodified reference itself ---------------------------------------------
needs_ref = pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")


@needs_ref
def test_workload_generator_matches_reference():
    for args in [(300, 5, 16, 16, 13), (1000, 3, 64, 1, 40000)]:
        a = O.generate_workload(*args)
        b = O.generate_workload(*args, use_ref=True)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))
    a = O.generate_workload(4096, 0, 64, 1, 40001, needle=True)
    b = O.generate_workload(4096, 0, 64, 1, 40001, needle=True, use_ref=True)
    assert all(np.array_equal(x, y) for x, y in zip(a, b))


@needs_ref
@pytest.mark.parametrize("cfg", [(16, 32, 128, 8, 4), (32, 64, 512, 8, 4), (16, 16, 64, 4, 2),
                                 (24, 32, 128, 16, 16), (20, 24, 96, 6, 3)])
def test_engine_bit_identical_to_reference(cfg):
    d, B, lf, kb, vb = cfg
    pk, pv, dk, dv, dq = O.generate_workload(900, 12, d, d, 5)
    e = O.OracleEngine(d, d, B, lf, kb, vb)
    r = O.RefEngine(lf * 2 * d * 2, d, d, B, kb, vb)
    assert r.l_fast() == lf
    e.prefill(pk, pv)
    r.prefill(pk, pv)
    for t in range(12):
        x = e.decode_step(dq[t], dk[t], dv[t])
        y = r.decode_step(dq[t], dk[t], dv[t])
        assert np.array_equal(x["output"][0], y["output"])  # bit-identical fp64
        assert np.array_equal(x["fetched"][0], y["fetched"])
        assert x["bytes_transferred"] == y["bytes_transferred"]
        assert x["eviction_occurred"] == y["eviction_occurred"]
    assert e.slow_blocks() == r.slow_blocks()
    for i in range(e.slow_blocks()):
        assert e.serialize_block(i) == r.serialize_block(i)


@needs_ref
def test_literal_merge_bit_identical_to_reference():
    # EngineOptions::literal_additive_merge (engine.cpp:44-48, 67-72)
    pk, pv, dk, dv, dq = O.generate_workload(512, 6, 16, 16, 13)
    e = O.OracleEngine(16, 16, 32, 128, 8, 4, None, 0.45)
    r = O.RefEngine(128 * 32 * 2, 16, 16, 32, 8, 4, literal_merge=True)
    e.prefill(pk, pv)
    r.prefill(pk, pv)
    for t in range(6):
        x = e.decode_step(dq[t], dk[t], dv[t], mode=2)
        y = r.decode_step(dq[t], dk[t], dv[t])
        assert np.array_equal(x["output"][0], y["output"])


@needs_ref
def test_quantize_bit_identical_to_reference():
    rng = np.random.default_rng(2)
    for trial in range(40):
        rows, dk, dv = int(rng.integers(1, 64)), int(rng.integers(1, 40)), int(rng.integers(1, 40))
        kb = int(rng.choice([2, 3, 4, 5, 6, 7, 8, 16]))
        vb = int(rng.choice([b for b in [2, 3, 4, 5, 6, 7, 8, 16] if b <= kb]))
        k = (rng.standard_normal((rows, dk)) * 3).astype(np.float32)
        v = rng.standard_normal((rows, dv)).astype(np.float32)
        n = O.ref().ref_quantize_serialize(k.reshape(-1), v.reshape(-1), rows, dk, dv, kb, vb, 7,
                                           100, None, 0)
        import ctypes as C
        buf = (C.c_uint8 * n)()
        O.ref().ref_quantize_serialize(k.reshape(-1), v.reshape(-1), rows, dk, dv, kb, vb, 7, 100,
                                       buf, n)
        kp, pk = O.quantize_tensor(k, kb)
        vp, pvv = O.quantize_tensor(v, vb)
        cen = np.zeros(dk, np.float32)
        O.oracle().tko_centroid(k.reshape(-1), rows, dk, cen)
        m = O.oracle().tko_serialize_block
        mine = (C.c_uint8 * n)()
        m.restype = C.c_size_t
        got = m(C.c_uint64(7), C.c_uint64(100), C.c_uint64(100 + rows - 1), C.c_uint32(rows),
                C.c_uint32(dk), C.c_uint32(dv), C.c_uint(kb), C.c_uint(vb),
                kp.ctypes.data_as(C.c_void_p), vp.ctypes.data_as(C.c_void_p),
                cen.ctypes.data_as(C.c_void_p), pk.ctypes.data_as(C.c_void_p),
                pvv.ctypes.data_as(C.c_void_p), mine)
        assert got == n and bytes(mine) == bytes(buf)


@needs_ref
def test_reference_criterion3_through_harness():
    import ctypes as C
    tot = C.c_uint64()
    ratio = O.ref().ref_traffic_reduction(C.byref(tot))
    assert tot.value == 11238400
    assert abs(ratio - 5.638997722095672) < 1e-12
