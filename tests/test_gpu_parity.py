"""GPU parity: libttkv_gpu.so (through the C ABI) vs the CPU oracle.

Contract (BASELINE.json north_star):
  * quantization codes, scales, centroids and the serialized block layout are
    bit-exact (serialize_block bytes equal, quantizer.cpp:248-274);
  * selected slow-tier block lists are identical, in schedule order;
  * bytes_transferred (modeled) and eviction reports are identical;
  * attention outputs are within 1e-3 relative L2 (reference.cpp:43-51) of the
    oracle's fp64 engine -- fp32 accumulation on the GPU.
Inputs for fp16 rings are rounded to fp16 first; fp32
rings (bytes_full_precision=4) take arbitrary floats.
"""
import numpy as np
import pytest

import _oracle as O

pytestmark = pytest.mark.gpu

OUT_TOL = 1e-3


def rel_err(a, b):
    a = np.asarray(a, np.float64).ravel()
    b = np.asarray(b, np.float64).ravel()
    den = np.sqrt((b * b).sum())
    return np.sqrt(((a - b) ** 2).sum()) / (den if den > 0 else 1.0)


# ---------------------------------------------------------------------------
# stateless quantize_block (quantizer.cpp:126-155)
# ---------------------------------------------------------------------------
def gpu_quantize(T, keys, values, kb, vb):
    import ctypes as C
    from paper_2604_19769_b200 import _lib as L
    keys = np.ascontiguousarray(keys, np.float32)
    values = np.ascontiguousarray(values, np.float32)
    rows, dk = keys.shape
    dv = values.shape[1]
    pk = np.zeros(max(1, T.packed_bytes(rows * dk, kb)), np.uint8)
    pv = np.zeros(max(1, T.packed_bytes(rows * dv, vb)), np.uint8)
    kp = np.zeros(2 * dk, np.float32)
    vp = np.zeros(2 * dv, np.float32)
    cen = np.zeros(dk, np.float32)
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    rc = L.lib().ttkv_gpu_quantize_block(0, p(keys), p(values), rows, dk, dv, kb, vb, p(pk),
                                         p(pv), p(kp), p(vp), p(cen))
    assert rc == 0, L.lib().ttkv_last_error()
    return pk[:T.packed_bytes(rows * dk, kb)], pv[:T.packed_bytes(rows * dv, vb)], kp, vp, cen


def test_golden_4bit_packing(gpu):
    # test_quantizer.cpp:36-52
    pk, pv, kp, vp, cen = gpu_quantize(gpu, np.array([[0.], [5.], [10.], [15.]]),
                                       np.full((4, 1), 2.0), 4, 4)
    assert list(pk) == [0x50, 0xFA]
    assert kp[0] == 1.0 and kp[1] == 0.0


def test_golden_2bit_packing(gpu):
    # test_quantizer.cpp:54-66
    pk, *_ = gpu_quantize(gpu, np.array([[1.], [2.], [3.], [0.], [3.]]), np.zeros((5, 1)), 2, 2)
    assert list(pk) == [0x39, 0x03]


def test_constant_channels(gpu):
    # test_quantizer.cpp:68-81
    k = np.tile(np.array([-4.25, 0.0, 1e-20], np.float32), (16, 1))
    v = np.tile(np.array([123.5, -0.125], np.float32), (16, 1))
    pk, pv, kp, vp, cen = gpu_quantize(gpu, k, v, 8, 4)
    back = O.dequantize_tensor(pk, 16, 3, 8, kp)
    assert np.array_equal(back, k)
    assert np.array_equal(O.dequantize_tensor(pv, 16, 2, 4, vp), v)


def test_centroid_is_prequant_mean(gpu):
    # test_quantizer.cpp:145-152
    k = np.array([[1, 0], [2, 4], [3, 0], [6, 4]], np.float32)
    *_, cen = gpu_quantize(gpu, k, np.zeros((4, 1)), 4, 4)
    assert cen[0] == 3.0 and cen[1] == 2.0


@pytest.mark.parametrize("bits", [(8, 4), (8, 8), (4, 4), (2, 2), (3, 2), (5, 3), (7, 7),
                                  (16, 16), (16, 4), (6, 5)])
def test_quantize_matches_oracle_bitexact(gpu, bits):
    kb, vb = bits
    rng = np.random.default_rng(kb * 10 + vb)
    for trial in range(12):
        rows = int(rng.choice([1, 3, 4, 24, 32, 128, 256]))
        dk = int(rng.integers(1, 129))
        dv = int(rng.integers(1, 129))
        scale = float(rng.choice([1e-3, 1.0, 50.0]))
        k = (rng.standard_normal((rows, dk)) * scale).astype(np.float32)
        v = (rng.uniform(-4, 4, (rows, dv))).astype(np.float32)
        if trial % 4 == 0:
            k[:, 0] = 1.5  # constant channel
        pk, pv, kp, vp, cen = gpu_quantize(gpu, k, v, kb, vb)
        okp, opk = O.quantize_tensor(k, kb)
        ovp, opv = O.quantize_tensor(v, vb)
        ocen = np.zeros(dk, np.float32)
        O.oracle().tko_centroid(k.reshape(-1), rows, dk, ocen)
        assert pk.tobytes() == opk.tobytes(), (rows, dk, kb)
        assert pv.tobytes() == opv.tobytes(), (rows, dv, vb)
        if kb != 16:
            assert kp.tobytes() == okp.tobytes()
        if vb != 16:
            assert vp.tobytes() == ovp.tobytes()
        assert cen.tobytes() == ocen.tobytes()


@pytest.mark.parametrize("bits", [(8, 4), (4, 2), (3, 3)])
def test_quantize_exact_half_ties(gpu, bits):
    # (x - lo) / scale landing exactly on k + 0.5: quantizer.cpp:82 rounds half
    # away from zero; the GPU takes its exact-division path for these elements
    kb, vb = bits
    rng = np.random.default_rng(kb + 17 * vb)
    rows = 128

    def tied(levels, dim):
        step = np.float32(rng.choice([1.0, 0.5, 0.25, 2.0]))
        x = (rng.integers(0, 2 * levels + 1, (rows, dim)).astype(np.float32) * np.float32(0.5)
             * step)
        x[0, :] = 0.0
        x[1, :] = np.float32(levels) * step  # lo = 0, hi = levels * step -> scale = step
        return x

    k, v = tied((1 << kb) - 1, 64), tied((1 << vb) - 1, 48)
    pk, pv, kp, vp, cen = gpu_quantize(gpu, k, v, kb, vb)
    okp, opk = O.quantize_tensor(k, kb)
    ovp, opv = O.quantize_tensor(v, vb)
    assert pk.tobytes() == opk.tobytes()
    assert pv.tobytes() == opv.tobytes()
    assert kp.tobytes() == okp.tobytes() and vp.tobytes() == ovp.tobytes()


# ---------------------------------------------------------------------------
# engine parity
# ---------------------------------------------------------------------------
def make_inputs(S, ctx, T, dk, dv, G, seed, fp16):
    """Reference workload per stream (workload.cpp:42-95), seed = base + s; the
    extra GQA queries come from the same generator family."""
    pk, pv, dkk, dvv, dq = [], [], [], [], []
    for s in range(S):
        a, b, c, d, q = O.generate_workload(max(ctx, 1), T, dk, dv, seed + s)
        a, b = a[:ctx], b[:ctx]  # ctx == 0: decode from an empty store
        qs = [q]
        for g in range(1, G):
            *_, qg = O.generate_workload(1, T, dk, dv, 7919 * (seed + s) + g)
            qs.append(qg)
        pk.append(a); pv.append(b); dkk.append(c); dvv.append(d)
        dq.append(np.stack(qs, axis=1))  # [T, G, dk]
    pk, pv, dkk, dvv, dq = map(np.stack, (pk, pv, dkk, dvv, dq))
    if fp16:
        pk, pv, dkk, dvv = map(O.fp16_round, (pk, pv, dkk, dvv))
    return pk, pv, dkk, dvv, dq  # dq: [S, T, G, dk]


def check_streamed_sets(eng, s, expected, G):
    """The GPU's own selection (ttkv_gpu_read_selected / read_union: the
    records the slow kernel streamed) equals `expected[g]` as a set for every
    head, and the per-stream union is exactly their union with the right head
    bits (relevance.cpp:29-43; each record streamed once)."""
    want = {}
    for g in range(G):
        exp = np.sort(np.asarray(expected[g], np.int64))
        got = eng.read_selected(s, g).astype(np.int64)
        assert np.array_equal(got, exp), (s, g, len(got), len(exp))
        for b in exp:
            want[int(b)] = want.get(int(b), 0) | (1 << g)
    ids, masks = eng.read_union(s)
    assert list(ids) == sorted(want), s
    assert [int(m) for m in masks] == [want[int(b)] for b in ids], s


def host_top_k(scores, k):
    """select_top_k (relevance.cpp:29-43) on the host: score desc, id desc."""
    ids = np.arange(len(scores), dtype=np.int64)
    order = np.lexsort((-ids, -np.asarray(scores, np.float64)))
    return order[:k]


def check_every_list(eng, S, G, k):
    """Every (stream, head) list the GPU streamed equals the top-k of the
    step's bit-exact device scores taken on the host; returns the union size."""
    union = 0
    for s in range(S):
        exp = [host_top_k(eng.read_scores(s, g), k) for g in range(G)]
        for g in range(G):
            assert np.array_equal(eng.read_fetched(s, g).astype(np.int64), exp[g]), (s, g)
        check_streamed_sets(eng, s, exp, G)
        union += len(set(np.concatenate(exp).tolist()))
    return union


def run_parity(T_, *, S=2, G=1, d=32, dv=None, B=32, l_fast=128, kb=8, vb=4, elem=2, ctx=600,
               steps=6, frac=0.45, top_k=None, mode=0, seed=100, prefill_chunks=1,
               check_blocks=True, literal=False, slow_tier=0, q_mul=1.0, kv_mul=1.0,
               record_stream=0):
    dv = dv or d
    cfg = T_.TierConfig(hbm_budget_bytes=l_fast * (d + dv) * elem, d_k=d, d_v=dv,
                        bytes_full_precision=elem, block_size=B, key_bits=kb, value_bits=vb,
                        fetch_fraction=frac, top_k_blocks=top_k)
    pol = T_.SelectionPolicy(top_k, frac)
    assert T_.fast_capacity(cfg) == l_fast
    pk, pv, dk_, dv_, dq = make_inputs(S, ctx, steps, d, dv, G, seed, fp16=(elem == 2))
    if q_mul != 1.0 or kv_mul != 1.0:
        dq = (dq * q_mul).astype(np.float32)
        pk, pv, dk_, dv_ = ((x * kv_mul).astype(np.float32) for x in (pk, pv, dk_, dv_))
        if elem == 2:
            pk, pv, dk_, dv_ = map(O.fp16_round, (pk, pv, dk_, dv_))
    eng = T_.MultiStreamEngine(cfg, pol, n_streams=S, heads_per_stream=G, group_select=bool(mode),
                               literal_additive_merge=literal, slow_tier=slow_tier,
                               record_stream=record_stream)
    orc = [O.OracleEngine(d, dv, B, l_fast, kb, vb, top_k, frac) for _ in range(S)]
    bounds = np.linspace(0, ctx, prefill_chunks + 1).astype(int)
    for a, b in zip(bounds[:-1], bounds[1:]):
        if b > a:
            eng.prefill(pk[:, a:b], pv[:, a:b])
    for s in range(S):
        if ctx:
            orc[s].prefill(pk[s], pv[s])
    st = eng.state()
    assert st["slow_blocks"] == orc[0].slow_blocks()
    assert st["fast_tokens"] == orc[0].fast_tokens()
    worst = 0.0
    for t in range(steps):
        rep = eng.decode_step(dq[:, t], dk_[:, t], dv_[:, t], fetched=True)
        for s in range(S):
            o = orc[s].decode_step(dq[s, t], dk_[s, t], dv_[s, t], mode=mode | (2 * literal))
            assert rep.blocks_scored == o["blocks_scored"]
            assert rep.eviction_occurred == o["eviction_occurred"]
            assert rep.bytes_transferred == o["bytes_transferred"]
            check_streamed_sets(eng, s, o["fetched"], G)
            for g in range(G):
                assert np.array_equal(rep.fetched_blocks[s][g], o["fetched"][g]), (t, s, g)
                e = rel_err(rep.output[s, g], o["output"][g])
                worst = max(worst, e)
                # fp16 ring: fp32 accumulation (north star 1e-3); fp32 ring: fp64
                assert e < (OUT_TOL if elem == 2 else 1e-9), (t, s, g, e)
    st = eng.state()
    assert st["slow_blocks"] == orc[0].slow_blocks()
    assert st["fast_tokens"] == orc[0].fast_tokens()
    if check_blocks:
        for s in range(S):
            for b in range(orc[s].slow_blocks()):
                assert eng.serialize_block(s, b) == orc[s].serialize_block(b), (s, b)
    eng.close()
    return worst


@pytest.mark.parametrize("ctx", [70000, 140000])
def test_engine_many_blocks_selection(gpu, ctx):
    # n = 4371 / 8746 slow blocks per stream: the radix select with its order
    # keys cached in shared memory (n <= 5632) and uncached (re-read from L2
    # every pass); the streamed sets are read back and compared exactly
    run_parity(gpu, S=2, G=2, d=16, B=16, l_fast=64, ctx=ctx, steps=2, check_blocks=False)


@pytest.mark.parametrize("elem", [4, 2])
def test_engine_uncached_radix_select_d128(gpu, elem):
    # d = 128 with n = 6234 > kTopkSmemKeys (5632): the uncached radix path at
    # the hot head dimension; fp32 ring -> outputs to 1e-9, so one wrongly
    # streamed block could not hide under the tolerance either
    run_parity(gpu, S=2, G=4, d=128, B=16, l_fast=256, ctx=100000, steps=2, elem=elem,
               check_blocks=False)


def test_engine_reference_unit_config(gpu):
    # test_engine.cpp:18-37 shape: d=16, B=32, 128-token fast tier, 512 ctx
    run_parity(gpu, S=1, G=1, d=16, B=32, l_fast=128, ctx=512, steps=6, seed=13)


def test_engine_fp32_ring_arbitrary_floats(gpu):
    run_parity(gpu, S=3, G=1, d=16, B=32, l_fast=128, ctx=512, steps=8, elem=4)


@pytest.mark.parametrize("bits", [(8, 4), (8, 8), (4, 4), (4, 2), (16, 16), (3, 3)])
def test_engine_bit_widths(gpu, bits):
    run_parity(gpu, S=2, G=2, d=32, B=32, l_fast=128, ctx=700, steps=5, kb=bits[0], vb=bits[1])


def test_engine_gqa_per_head(gpu):
    run_parity(gpu, S=3, G=4, d=64, B=64, l_fast=256, ctx=2000, steps=6)


def test_engine_gqa_group_shared(gpu):
    run_parity(gpu, S=3, G=4, d=64, B=64, l_fast=256, ctx=2000, steps=6, mode=1)


def test_engine_literal_additive_merge(gpu):
    # EngineOptions::literal_additive_merge (engine.cpp:44-48, 67-72)
    run_parity(gpu, S=2, G=2, d=16, B=32, l_fast=128, ctx=600, steps=4, literal=True)
    run_parity(gpu, S=2, G=4, d=64, B=64, l_fast=256, ctx=2000, steps=3, literal=True, mode=1)


def test_engine_eviction_cycle(gpu):
    # crosses several eviction steps (fast tier cycles l_fast+1 -> l_fast-B+1)
    run_parity(gpu, S=2, G=2, d=16, B=16, l_fast=64, ctx=300, steps=40)


def test_engine_ragged_dims(gpu):
    run_parity(gpu, S=2, G=3, d=20, dv=7, B=24, l_fast=96, ctx=333, steps=6, kb=6, vb=3)


def test_engine_context_shorter_than_fast_tier(gpu):
    run_parity(gpu, S=2, G=1, d=16, B=32, l_fast=128, ctx=50, steps=4)


def test_engine_empty_prefill(gpu):
    run_parity(gpu, S=1, G=2, d=16, B=16, l_fast=32, ctx=0, steps=40)


def test_engine_top_k_absolute_and_zero(gpu):
    run_parity(gpu, S=2, G=1, d=16, B=32, l_fast=128, ctx=800, steps=3, top_k=5)
    run_parity(gpu, S=2, G=1, d=16, B=32, l_fast=128, ctx=800, steps=3, top_k=0)
    run_parity(gpu, S=2, G=1, d=16, B=32, l_fast=128, ctx=800, steps=3, top_k=1000)


def test_engine_fetch_all(gpu):
    run_parity(gpu, S=2, G=2, d=32, B=32, l_fast=128, ctx=900, steps=3, frac=1.0)


def test_engine_chunked_prefill(gpu):
    run_parity(gpu, S=2, G=1, d=16, B=32, l_fast=128, ctx=1000, steps=3, prefill_chunks=7)


def test_engine_hot_shape_small(gpu):
    # the hot-path shape (d=128, B=128, K8/V4, G=4) at a small context
    run_parity(gpu, S=4, G=4, d=128, B=128, l_fast=1024, ctx=6000, steps=4, check_blocks=True)


@pytest.mark.parametrize("G,mode,literal", [(4, 0, False), (4, 1, False), (1, 0, False), (2, 0, False),
                                            (3, 0, False), (6, 0, False), (5, 1, False),
                                            (8, 0, False), (4, 0, True)])
@pytest.mark.parametrize("record_stream", [1, 2])
def test_engine_hbm_resident_slow_tier(gpu, G, mode, literal, record_stream):
    # slow tier in HBM: the tensor-core slow kernel (TMA tensor maps, mma.sync
    # on raw codes) for K8/V4, d = B = 128; records still bit-exact.  Both
    # record streams: the selected union after the selection (1) and the
    # speculative stream of every record beside it (2, G <= 4 and not literal;
    # otherwise the handle keeps the union stream)
    run_parity(gpu, S=3, G=G, d=128, B=128, l_fast=512, ctx=5000, steps=4, mode=mode,
               literal=literal, slow_tier=1, record_stream=record_stream)


@pytest.mark.parametrize("slow_tier,record_stream", [(0, 0), (1, 1), (1, 2)])
@pytest.mark.parametrize("q_mul,kv_mul", [(3e4, 1.0), (1.0, 2e3), (50.0, 2e3), (1e-6, 1e-3), (1e7, 1.0), (3e3, 5e3)])
def test_engine_extreme_magnitudes(gpu, slow_tier, record_stream, q_mul, kv_mul):
    # hot-path shape with queries / KV far from N(0, 1): the tensor-core
    # kernels' fp16 operand splits must neither overflow (scores of 1e4+ in
    # log2 units, keys near the fp16 range) nor lose the small end
    run_parity(gpu, S=2, G=4, d=128, B=128, l_fast=512, ctx=3000, steps=3, slow_tier=slow_tier,
               q_mul=q_mul, kv_mul=kv_mul, record_stream=record_stream)


@pytest.mark.parametrize("slow_tier,record_stream", [(0, 0), (1, 1), (1, 2)])
def test_engine_long_fast_tier_short_slow(gpu, slow_tier, record_stream):
    # a long fast tier (second stream) against a one-record slow tier: the
    # combine, launched chained behind the short slow kernel, must still wait
    # for the fast tier's event (programmatic launch must not bypass it)
    run_parity(gpu, S=4, G=4, d=128, B=128, l_fast=16384, ctx=16384 + 200, steps=4,
               slow_tier=slow_tier, check_blocks=False, record_stream=record_stream)


def test_engine_hbm_resident_generic_shape(gpu):
    # a shape the tensor-core kernel does not cover -> CUDA-core slow kernel on HBM
    run_parity(gpu, S=2, G=2, d=32, B=32, l_fast=128, ctx=900, steps=4, slow_tier=1)


def test_lossless_fetch_all_matches_dense(gpu):
    # test_engine.cpp:35-48: 16/16 + fetch-all == dense attention (fp32 ring)
    T_ = gpu
    d, B, lf, ctx, steps = 16, 32, 128, 512, 6
    cfg = T_.TierConfig(hbm_budget_bytes=lf * 2 * d * 4, d_k=d, d_v=d, bytes_full_precision=4,
                        block_size=B, key_bits=16, value_bits=16, fetch_fraction=1.0)
    pk, pv, dk_, dv_, dq = O.generate_workload(ctx, steps, d, d, 13)
    eng = T_.Engine(cfg, T_.SelectionPolicy(None, 1.0))
    eng.prefill(pk, pv)
    hk, hv = list(pk), list(pv)
    for t in range(steps):
        r = eng.decode_step(dq[t], dk_[t], dv_[t])
        hk.append(dk_[t]); hv.append(dv_[t])
        dense = np.zeros(d, np.float64)
        O.oracle().tko_dense_attention(dq[t], d, np.ascontiguousarray(hk).reshape(-1),
                                       np.ascontiguousarray(hv).reshape(-1), len(hk), d, dense)
        assert rel_err(r.output, dense) < 1e-12  # fp32 ring -> fp64 accumulation
        assert r.blocks_fetched == r.blocks_scored
    eng.close()


def test_store_state_and_locate(gpu):
    # test_tier_store.cpp:48-81 semantics through the GPU store
    T_ = gpu
    cfg = T_.TierConfig(hbm_budget_bytes=8 * 8 * 2, d_k=4, d_v=4, block_size=4)
    eng = T_.MultiStreamEngine(cfg, n_streams=1)
    assert eng.state()["l_fast"] == 8
    toks = np.array([[p] * 4 for p in range(9)], np.float32)
    eng.prefill(toks[None], (toks * 0.5)[None])
    st = eng.state()
    assert st["fast_tokens"] == 5 and st["slow_blocks"] == 1
    for p in range(4):
        assert eng.locate(p) == ("slow", 0)
    for p in range(4, 9):
        assert eng.locate(p)[0] == "fast"
    assert eng.locate(9)[0] == "absent"
    blk = eng.read_block(0, 0)
    back = O.dequantize_tensor(blk["packed_keys"], 4, 4, 8, blk["key_params"])
    assert abs(back[0, 0] - 0.0) < 1e-6 and abs(back[3, 0] - 3.0) < 1e-6
    k, v, first = eng.read_fast(0)
    assert first == 4 and np.array_equal(k[:, 0], np.arange(4, 9, dtype=np.float32))
    eng.close()


def test_dump_slow_tier_byte_identical(gpu, tmp_path):
    T_ = gpu
    d, B, lf = 16, 16, 64
    cfg = T_.TierConfig(hbm_budget_bytes=lf * 2 * d * 2, d_k=d, d_v=d, block_size=B)
    pk, pv, *_ = O.generate_workload(400, 1, d, d, 5)
    pk, pv = O.fp16_round(pk), O.fp16_round(pv)
    eng = T_.MultiStreamEngine(cfg, n_streams=1)
    eng.prefill(pk[None], pv[None])
    orc = O.OracleEngine(d, d, B, lf)
    orc.prefill(pk, pv)
    path = tmp_path / "tier.bin"
    eng.dump_slow_tier(0, path)
    n = orc.slow_blocks()
    expect = b"TTKVTIER" + (1).to_bytes(2, "little") + n.to_bytes(8, "little")
    for b in range(n):
        blob = orc.serialize_block(b)
        expect += len(blob).to_bytes(8, "little") + blob
    assert path.read_bytes() == expect
    eng.close()


def test_errors_map_to_reference_classes(gpu):
    T_ = gpu
    with pytest.raises(T_.ConfigError):
        T_.MultiStreamEngine(T_.TierConfig(hbm_budget_bytes=100, d_k=16, d_v=16))
    with pytest.raises(T_.ConfigError):
        T_.MultiStreamEngine(T_.TierConfig(hbm_budget_bytes=1 << 20, d_k=16, d_v=16,
                                           key_bits=4, value_bits=8))
    cfg = T_.TierConfig(hbm_budget_bytes=1 << 16, d_k=16, d_v=16)
    eng = T_.MultiStreamEngine(cfg)
    with pytest.raises(T_.ShapeError):
        eng.decode_step(np.zeros(7, np.float32), np.zeros(16, np.float32),
                        np.zeros(16, np.float32))
    eng.close()


# ---------------------------------------------------------------------------
# the unmodified reference (oracle/_ref) as the second checker
# ---------------------------------------------------------------------------
@pytest.mark.skipif(not O.ref_available(), reason="oracle/_ref not built")
def test_gpu_vs_reference_engine_fp32_ring(gpu):
    """Criterion-3 operating point (acceptance.cpp:172-195): seed 3, 16K ctx,
    1024-token fast tier, K8/V4, 0.45, 8 steps.  fp32 ring -> bit-exact
    selection against the reference itself, and the reference's own golden
    H->G total of 11,238,400 B."""
    T_ = gpu
    d, B, lf, ctx, steps = 128, 128, 1024, 16384, 8
    pk, pv, dk_, dv_, dq = O.generate_workload(ctx, steps, d, d, 3, use_ref=True)
    cfg = T_.TierConfig(hbm_budget_bytes=lf * 256 * 4, d_k=d, d_v=d, bytes_full_precision=4,
                        block_size=B)
    eng = T_.Engine(cfg, T_.SelectionPolicy(None, 0.45))
    ref = O.RefEngine(lf * 256 * 2, d, d, B)
    eng.prefill(pk, pv)
    ref.prefill(pk, pv)
    total = 0.0
    for t in range(steps):
        r = eng.decode_step(dq[t], dk_[t], dv_[t])
        o = ref.decode_step(dq[t], dk_[t], dv_[t])
        assert np.array_equal(r.fetched_blocks, o["fetched"])
        assert r.bytes_transferred == o["bytes_transferred"]
        assert rel_err(r.output, o["output"]) < OUT_TOL
        total += r.bytes_transferred
    assert total == 11238400.0
    for b in range(ref.slow_blocks()):
        assert eng.store.serialize_block(0, b) == ref.serialize_block(b)
    eng.close()


# ---------------------------------------------------------------------------
# full-size properties (cfg1 shape) with device-generated KV
# ---------------------------------------------------------------------------
def full_size_step(eng, q, kn, vn, sampled, k, B, d, kb=8, vb=4):
    """One decode step at a full BASELINE shape, checked three ways
    (engine.cpp:22-93):
      * sampled streams re-derived on the host from the read-back fast tier +
        records: fp64 scores bit-equal to the device's, every head's fetched
        list identical in order to select_top_k's, the output within 1e-3 of an
        fp64 recomputation over exactly the selected blocks;
      * the record evicted at the end of the step equals the oracle's
        quantize_block of the fast-tier rows it came from (bit-exact);
      * every (stream, head) set the slow kernel streamed equals the host
        top-k of that head's device scores, and the per-step union matches the
        reported union / PCIe bytes."""
    S, G = q.shape[0], q.shape[1]
    st0 = eng.state()
    n = st0["slow_blocks"]
    before = {s: (eng.read_fast(s), [eng.read_block(s, b) for b in range(n)]) for s in sampled}
    rep = eng.decode_step(q, kn, vn, fetched=True)
    assert rep.blocks_scored == n and rep.blocks_fetched == k
    for s in sampled:
        (fk, fv, first), blocks = before[s]
        dk = [O.dequantize_tensor(b["packed_keys"], B, d, kb, b["key_params"]) for b in blocks]
        dv = [O.dequantize_tensor(b["packed_values"], B, d, vb, b["value_params"]) for b in blocks]
        for g in range(G):
            scores = np.array([O.oracle().tko_score_block(q[s, g], b["key_centroid"], d)
                               for b in blocks])
            assert np.array_equal(eng.read_scores(s, g), scores), (s, g)
            sel = np.zeros(k, np.uint64)
            O.oracle().tko_select_top_k(scores, None, n, k, sel)
            assert np.array_equal(rep.fetched_blocks[s][g], sel), (s, g)
            assert np.array_equal(eng.read_selected(s, g), np.sort(sel)), (s, g)
            K = np.concatenate([fk.astype(np.float64), kn[s][None].astype(np.float64)] +
                               [dk[int(b)] for b in sel])
            V = np.concatenate([fv.astype(np.float64), vn[s][None].astype(np.float64)] +
                               [dv[int(b)] for b in sel])
            lg = K @ q[s, g].astype(np.float64) / np.sqrt(d)
            w = np.exp(lg - lg.max())
            ref = (w[:, None] * V).sum(0) / w.sum()
            assert rel_err(rep.output[s, g], ref) < OUT_TOL, (s, g)
        if rep.eviction_occurred:
            # tier_store.cpp:71-98: the oldest B fast tokens become block n
            blk = eng.read_block(s, n)
            assert blk["first_position"] == first
            okp, opk = O.quantize_tensor(fk[:B], kb)
            ovp, opv = O.quantize_tensor(fv[:B], vb)
            ocen = np.zeros(d, np.float32)
            O.oracle().tko_centroid(np.ascontiguousarray(fk[:B]).reshape(-1), B, d, ocen)
            assert blk["packed_keys"].tobytes() == opk.tobytes(), s
            assert blk["packed_values"].tobytes() == opv.tobytes(), s
            assert blk["key_params"].tobytes() == okp.tobytes(), s
            assert blk["value_params"].tobytes() == ovp.tobytes(), s
            assert blk["key_centroid"].tobytes() == ocen.tobytes(), s
    union = check_every_list(eng, S, G, k)
    assert rep.union_blocks == union
    assert rep.pcie_bytes == union * eng.state()["payload_bytes"]
    return rep


def step_inputs(rng, S, G, d):
    q = rng.standard_normal((S, G, d)).astype(np.float32)
    kn = O.fp16_round(rng.standard_normal((S, d)))
    vn = O.fp16_round(rng.standard_normal((S, d)))
    return q, kn, vn


def test_full_size_cfg1_sampled_streams(gpu):
    """cfg1: 32 MHA streams, 32K ctx, 4K fp16 fast tier, K8/V4, 0.45 (n = 224,
    k = 101).  KV is generated on device; the step evicts one block per stream."""
    T_ = gpu
    S, d, B, lf, ctx = 32, 128, 128, 4096, 32768
    cfg = T_.TierConfig(hbm_budget_bytes=lf * 256 * 2, d_k=d, d_v=d, block_size=B)
    eng = T_.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=1, reserve_tokens=ctx + 256)
    eng.prefill_synthetic(ctx, seed=11)
    assert eng.state()["slow_blocks"] == 224
    rep = full_size_step(eng, *step_inputs(np.random.default_rng(0), S, 1, d), (0, S - 1), 101, B, d)
    assert rep.eviction_occurred
    # every record streamed exactly once per step: union == k for G=1
    assert rep.union_blocks == S * 101
    eng.close()


@pytest.mark.parametrize("slow_tier", [0, 1])
def test_full_size_cfg2_sampled_streams(gpu, slow_tier):
    """cfg2 at full size: 256 streams (32 layers x 8 KV heads) x 4 query heads,
    128K ctx, 4K fp16 fast tier, K8/V4, 0.45 per query head (n = 992 blocks,
    k = 447), slow tier in pinned DRAM (CUDA-core streaming kernel) or HBM
    (tensor-core kernel); all 1024 streamed sets checked."""
    T_ = gpu
    S, G, d, B, lf, ctx = 256, 4, 128, 128, 4096, 131072
    cfg = T_.TierConfig(hbm_budget_bytes=lf * 256 * 2, d_k=d, d_v=d, block_size=B)
    eng = T_.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, reserve_tokens=ctx + 256,
                               slow_tier=slow_tier)
    eng.prefill_synthetic(ctx, seed=23)
    assert eng.state()["slow_blocks"] == 992
    rep = full_size_step(eng, *step_inputs(np.random.default_rng(1), S, G, d), (7, S - 3), 447,
                         B, d)
    assert rep.eviction_occurred
    eng.close()


@pytest.mark.parametrize("record_stream", [1, 2])
def test_full_size_cfg2_one_layer_hbm(gpu, record_stream):
    """One layer of cfg2 as layer-sequential decode runs it: 8 KV streams x 4
    query heads at 128K (n = 992, k = 447), slow tier in HBM, with the union
    record stream (1) and the speculative one (2: every record streamed beside
    the selection, the combine merging each head's selected records).  Every
    stream re-derived on the host, over steps that reuse the record queue."""
    T_ = gpu
    S, G, d, B, lf, ctx = 8, 4, 128, 128, 4096, 131072
    cfg = T_.TierConfig(hbm_budget_bytes=lf * 256 * 2, d_k=d, d_v=d, block_size=B)
    eng = T_.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, reserve_tokens=ctx + 256,
                               slow_tier=1, record_stream=record_stream)
    eng.prefill_synthetic(ctx, seed=29)
    rng = np.random.default_rng(9)
    for _ in range(3):
        full_size_step(eng, *step_inputs(rng, S, G, d), tuple(range(S)), 447, B, d)
    assert eng.state()["spec_steps"] == (3 if record_stream == 2 else 0)
    eng.close()


@pytest.mark.parametrize("slow_tier", [0, 1])
def test_full_size_cfg3_batch16(gpu, slow_tier):
    """cfg3 at full size: LLaMA-3-8B GQA at 32K ctx, batch 16 -> 4096 streams
    (32 layers x 8 KV heads x 16 requests) x 4 query heads (n = 224, k = 101):
    24 GB of records in pinned DRAM or HBM; all 16,384 streamed sets checked,
    three sampled streams (first request, middle, last) re-derived."""
    T_ = gpu
    S, G, d, B, lf, ctx = 4096, 4, 128, 128, 4096, 32768
    cfg = T_.TierConfig(hbm_budget_bytes=lf * 256 * 2, d_k=d, d_v=d, block_size=B)
    eng = T_.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, reserve_tokens=ctx + 256,
                               slow_tier=slow_tier)
    eng.prefill_synthetic(ctx, seed=31)
    assert eng.state()["slow_blocks"] == 224
    rep = full_size_step(eng, *step_inputs(np.random.default_rng(3), S, G, d), (0, 2053, S - 1),
                         101, B, d)
    assert rep.eviction_occurred
    eng.close()


@pytest.mark.parametrize("slow_tier", [0, 1])
def test_full_size_cfg5_256k_after_eviction_period(gpu, slow_tier):
    """cfg5 hot shape: 256 streams x 4 heads grown to 256K ctx through one full
    eviction period of decode (128 steps, the first evicting a block per
    stream into the slow tier), then the 128th step checked in full at
    n = 2016, k = 908 -- the scored slow tier includes the decode-time
    eviction's records."""
    T_ = gpu
    S, G, d, B, lf = 256, 4, 128, 128, 4096
    ctx0 = 262144 - 128
    cfg = T_.TierConfig(hbm_budget_bytes=lf * 256 * 2, d_k=d, d_v=d, block_size=B)
    eng = T_.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, reserve_tokens=262144 + 256,
                               slow_tier=slow_tier)
    eng.prefill_synthetic(ctx0, seed=47)
    assert eng.state()["slow_blocks"] == 2015
    rng = np.random.default_rng(5)
    # the first step evicts block 2015 from the fast tier: check it bit-exact
    rep = full_size_step(eng, *step_inputs(rng, S, G, d), (11,), 907, B, d)
    assert rep.eviction_occurred and eng.state()["slow_blocks"] == 2016
    for _ in range(126):
        rep = eng.decode_step(*step_inputs(rng, S, G, d))
        assert not rep.eviction_occurred and rep.blocks_fetched == 908
    assert eng.state()["appended"] == 262143
    rep = full_size_step(eng, *step_inputs(rng, S, G, d), (11, S - 1), 908, B, d)
    assert not rep.eviction_occurred and eng.state()["fast_tokens"] == 4096
    eng.close()


@pytest.mark.parametrize("slow_tier", [0, 1])
def test_host_api_pinned_buffers_direct(gpu, slow_tier):
    """ttkv_gpu_decode_step DMAs page-locked caller buffers directly (no
    staging copy) and writes the output into a page-locked `out`: the same
    steps through pageable and pinned buffers give bit-identical outputs and
    reports, across an eviction."""
    import torch
    T_ = gpu
    S, G, d, B, lf, ctx, steps = 3, 4, 128, 128, 512, 3000, 140
    cfg = T_.TierConfig(hbm_budget_bytes=lf * 2 * d * 2, d_k=d, d_v=d, block_size=B)
    rng = np.random.default_rng(17)
    pk = O.fp16_round(rng.standard_normal((S, ctx, d)))
    pv = O.fp16_round(rng.standard_normal((S, ctx, d)))
    ins = [(rng.standard_normal((S, G, d)).astype(np.float32),
            rng.standard_normal((S, d)).astype(np.float16),
            rng.standard_normal((S, d)).astype(np.float16)) for _ in range(steps)]

    def pinned(a):
        t = torch.empty(a.shape, dtype={np.float32: torch.float32, np.float16: torch.float16,
                                        np.float64: torch.float64}[a.dtype.type],
                        pin_memory=True)
        t.numpy()[...] = a
        return t
    runs = []
    for use_pinned in (False, True):
        eng = T_.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, slow_tier=slow_tier)
        eng.prefill(pk, pv)
        keep = []
        out_t = pinned(np.zeros((S, G, d), np.float64)) if use_pinned else None
        outs, evs = [], []
        for q, k, v in ins:
            if use_pinned:
                tq, tk, tv = pinned(q), pinned(k), pinned(v)
                keep += [tq, tk, tv]
                r = eng.decode_step(tq.numpy(), tk.numpy(), tv.numpy(), out=out_t.numpy())
                assert r.output is out_t.numpy() or np.shares_memory(r.output, out_t.numpy())
            else:
                r = eng.decode_step(q, k, v)
            outs.append(r.output.copy())
            evs.append((r.eviction_occurred, r.union_blocks, r.bytes_transferred))
        runs.append((np.stack(outs), evs))
        eng.close()
    assert np.array_equal(runs[0][0], runs[1][0])
    assert runs[0][1] == runs[1][1]
    assert any(e[0] for e in runs[0][1])


@pytest.mark.parametrize("dtype", ["f16", "f32"])
def test_prefill_from_device_memory(gpu, dtype):
    # ttkv_gpu_prefill_device reads the caller's [S][n][d] device rows in
    # place; records, fast tier and the next decode equal a host prefill's
    import torch
    T_ = gpu
    S, G, d, B, lf, ctx = 3, 2, 128, 128, 512, 5000
    cfg = T_.TierConfig(hbm_budget_bytes=lf * 2 * d * 2, d_k=d, d_v=d, block_size=B)
    rng = np.random.default_rng(4)
    pk = O.fp16_round(rng.standard_normal((S, ctx, d)))
    pv = O.fp16_round(rng.standard_normal((S, ctx, d)))
    host = T_.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G)
    host.prefill(pk, pv)
    dev = T_.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G)
    tdt = torch.float16 if dtype == "f16" else torch.float32
    tk = torch.from_numpy(pk).to("cuda", tdt).contiguous()
    tv = torch.from_numpy(pv).to("cuda", tdt).contiguous()
    dev.prefill_device(tk.data_ptr(), tv.data_ptr(), ctx, 1 if dtype == "f16" else 0)
    assert dev.state()["slow_blocks"] == host.state()["slow_blocks"]
    assert dev.state()["fast_tokens"] == host.state()["fast_tokens"]
    for s in range(S):
        for b in range(host.state()["slow_blocks"]):
            assert dev.serialize_block(s, b) == host.serialize_block(s, b)
    q = rng.standard_normal((S, G, d)).astype(np.float32)
    kn = O.fp16_round(rng.standard_normal((S, d)))
    vn = O.fp16_round(rng.standard_normal((S, d)))
    assert np.array_equal(dev.decode_step(q, kn, vn).output, host.decode_step(q, kn, vn).output)
    host.close()
    dev.close()


@pytest.mark.parametrize("slow_tier", [0, 1])
def test_engine_d64_tensor_core_fast_tier(gpu, slow_tier):
    # d = 64, B = 64: the tensor-core fast tier with one 64-channel box (ND = 1);
    # the slow tier takes the CUDA-core kernel (host DRAM or HBM)
    run_parity(gpu, S=3, G=4, d=64, B=64, l_fast=256, ctx=3000, steps=4, slow_tier=slow_tier)


@pytest.mark.parametrize("n", [1, 37, 8192, 8193, 20000, 70001])
def test_free_select_top_k_any_n(gpu, n):
    # the stateless select_top_k (relevance.cpp:29-43) on arbitrary ids and
    # heavily tied scores: shared-memory bitonic CTA up to 8192, global-memory
    # network above; order = score desc, id desc, for every k
    import ctypes as C
    from paper_2604_19769_b200 import _lib as L
    rng = np.random.default_rng(n)
    scores = np.round(rng.standard_normal(n) * 4) / 4  # many exact ties
    scores[rng.integers(0, n, max(1, n // 50))] = -0.0
    ids = rng.permutation(3 * n)[:n].astype(np.uint64)
    order = np.lexsort((-ids.astype(np.int64), -scores))
    p = lambda a: a.ctypes.data_as(C.c_void_p)
    for k in sorted({1, n // 3, n}):
        out = np.zeros(max(1, k), np.uint64)
        rc = L.lib().ttkv_gpu_select_top_k(0, p(scores), p(ids), n, k, p(out))
        assert rc == 0, L.lib().ttkv_last_error()
        assert np.array_equal(out[:k], ids[order[:k]]), (n, k)


@pytest.mark.parametrize("slow_tier", [0, 1])
def test_host_api_unaligned_buffers_match_device_path(gpu, slow_tier):
    """The host-buffer step's ingest kernel reads q/k/v through the device
    mapping of page-locked memory (16-byte accesses when aligned, bytes
    otherwise) and the combine writes the output there: page-locked buffers at
    odd offsets with a row size that is not a multiple of 16 bytes (d = 40,
    fp16 k/v) give the same bits as the device-buffer step on the same inputs,
    step after step (graph replays with changing addresses) across an eviction."""
    import torch
    T_ = gpu
    S, G, d, B, lf, ctx, steps = 3, 2, 40, 32, 256, 1000, 40
    cfg = T_.TierConfig(hbm_budget_bytes=lf * 2 * d * 2, d_k=d, d_v=d, block_size=B)
    rng = np.random.default_rng(23)
    pk = O.fp16_round(rng.standard_normal((S, ctx, d)))
    pv = O.fp16_round(rng.standard_normal((S, ctx, d)))
    ins = [(rng.standard_normal((S, G, d)).astype(np.float32),
            rng.standard_normal((S, d)).astype(np.float16),
            rng.standard_normal((S, d)).astype(np.float16)) for _ in range(steps)]
    keep = []

    def pinned_at(a, off):
        raw = torch.empty(a.nbytes + 64, dtype=torch.uint8, pin_memory=True)
        keep.append(raw)
        v = raw.numpy()[off:off + a.nbytes].view(a.dtype).reshape(a.shape)
        v[...] = a
        return v

    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    host = T_.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, slow_tier=slow_tier)
    devi = T_.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, slow_tier=slow_tier)
    devi.set_stream(stream.cuda_stream)
    for e in (host, devi):
        e.prefill(pk, pv)
    out_h = pinned_at(np.zeros((S, G, d), np.float64), 8)
    evicted = False
    for i, (q, k, v) in enumerate(ins):
        r = host.decode_step(pinned_at(q, 4 + 4 * (i % 3)), pinned_at(k, 2 + 2 * (i % 5)),
                             pinned_at(v, 6), out=out_h)
        evicted |= r.eviction_occurred
        tq, tk, tv = (torch.from_numpy(x).to(dev) for x in (q, k, v))
        to = torch.empty((S, G, d), dtype=torch.float64, device=dev)
        torch.cuda.synchronize()
        devi.decode_step_device(tq.data_ptr(), tk.data_ptr(), tv.data_ptr(), to.data_ptr())
        devi.synchronize()
        assert np.array_equal(out_h, to.cpu().numpy()), f"step {i}"
    assert evicted
    host.close()
    devi.close()
