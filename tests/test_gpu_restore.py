"""Checkpoint / resume of a GPU handle.

The reference persists the slow tier (dump_slow_tier / load_slow_tier,
quantizer.cpp:325-365) but cannot rebuild a TierStore from it
(tier_store.hpp:42).  ttkv_gpu_restore_slow_tier loads one TTKVTIER file per
stream into a fresh handle, the fast tier resumes through append, and decode
continues:
  * from files written by the UNMODIFIED reference (oracle/_ref serializes the
    blocks) the resumed GPU engine matches the reference engine that never
    stopped: fetched lists identical, outputs within 1e-3, every later
    evicted record byte-identical;
  * checkpoint() -> restore() of a GPU handle resumes bit-identically;
  * damaged or mismatched files fail with the reference's error classes.
"""
import numpy as np
import pytest

import _oracle as O

pytestmark = pytest.mark.gpu


def tier_file(blobs):
    """dump_slow_tier's container (quantizer.cpp:325-342) around serialized blocks."""
    out = b"TTKVTIER" + (1).to_bytes(2, "little") + len(blobs).to_bytes(8, "little")
    for b in blobs:
        out += len(b).to_bytes(8, "little") + b
    return out


def rel_err(a, b):
    a, b = np.asarray(a, np.float64).ravel(), np.asarray(b, np.float64).ravel()
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_resume_from_reference_dump(gpu, tmp_path):
    T = gpu
    S, d, B, lf, ctx, steps = 3, 64, 32, 256, 1500, 70
    rng = np.random.default_rng(3)
    pk = O.fp16_round(rng.standard_normal((S, ctx, d)))
    pv = O.fp16_round(rng.standard_normal((S, ctx, d)))
    refs = []
    paths = []
    for s in range(S):
        r = O.RefEngine(lf * 2 * d * 2, d, d, B)
        r.prefill(pk[s], pv[s])
        refs.append(r)
        p = tmp_path / f"s{s}.ttkvtier"
        p.write_bytes(tier_file([r.serialize_block(b) for b in range(r.slow_blocks())]))
        paths.append(p)
    n = refs[0].slow_blocks()
    cfg = T.TierConfig(hbm_budget_bytes=lf * 2 * d * 2, d_k=d, d_v=d, block_size=B)
    eng = T.MultiStreamEngine(cfg, n_streams=S)
    eng.restore_slow_tier(paths)
    assert eng.state()["slow_blocks"] == n and eng.state()["appended"] == n * B
    eng.append(pk[:, n * B:], pv[:, n * B:])  # the fast tier resumes
    assert eng.state()["fast_tokens"] == ctx - n * B
    for s in range(S):  # restored records serialize back to the reference's bytes
        for b in (0, n // 2, n - 1):
            assert eng.serialize_block(s, b) == refs[s].serialize_block(b)
    evicted = 0
    for t in range(steps):
        q = rng.standard_normal((S, 1, d)).astype(np.float32)
        kn = O.fp16_round(rng.standard_normal((S, d)))
        vn = O.fp16_round(rng.standard_normal((S, d)))
        rep = eng.decode_step(q, kn, vn, fetched=True)
        for s in range(S):
            o = refs[s].decode_step(q[s, 0], kn[s], vn[s])
            assert np.array_equal(rep.fetched_blocks[s][0], o["fetched"]), (t, s)
            assert rel_err(rep.output[s, 0], o["output"]) < 1e-3
            assert rep.bytes_transferred == o["bytes_transferred"]
        evicted += rep.eviction_occurred
    assert evicted >= 2  # blocks evicted after the resume
    for s in range(S):
        for b in range(n, refs[s].slow_blocks()):
            assert eng.serialize_block(s, b) == refs[s].serialize_block(b)
    eng.close()


@pytest.mark.parametrize("G,slow_tier", [(4, 0), (4, 1), (1, 0)])
def test_checkpoint_restore_bit_identical(gpu, tmp_path, G, slow_tier):
    T = gpu
    S, d, B, lf, ctx = 4, 128, 128, 512, 3000
    cfg = T.TierConfig(hbm_budget_bytes=lf * 2 * d * 2, d_k=d, d_v=d, block_size=B)
    rng = np.random.default_rng(9)
    pk = O.fp16_round(rng.standard_normal((S, ctx, d)))
    pv = O.fp16_round(rng.standard_normal((S, ctx, d)))
    a = T.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, slow_tier=slow_tier)
    a.prefill(pk, pv)

    def step_inputs(n):
        return [(rng.standard_normal((S, G, d)).astype(np.float32),
                 O.fp16_round(rng.standard_normal((S, d))),
                 O.fp16_round(rng.standard_normal((S, d)))) for _ in range(n)]

    for q, k, v in step_inputs(5):
        a.decode_step(q, k, v)
    a.checkpoint(tmp_path / "ckpt")
    b = T.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, slow_tier=slow_tier)
    b.restore(tmp_path / "ckpt")
    assert b.state()["appended"] == a.state()["appended"]
    assert b.state()["slow_blocks"] == a.state()["slow_blocks"]
    evictions = 0
    for q, k, v in step_inputs(140):  # crosses at least one eviction
        ra = a.decode_step(q, k, v, fetched=True)
        rb = b.decode_step(q, k, v, fetched=True)
        assert np.array_equal(ra.output, rb.output)
        assert all(np.array_equal(x, y) for fa, fb in zip(ra.fetched_blocks, rb.fetched_blocks)
                   for x, y in zip(fa, fb))
        evictions += ra.eviction_occurred
    assert evictions >= 1
    for s in range(S):
        for blk in range(a.state()["slow_blocks"]):
            assert a.serialize_block(s, blk) == b.serialize_block(s, blk)
    a.close()
    b.close()


def test_restore_errors(gpu, tmp_path):
    T = gpu
    d, B, lf = 16, 16, 64
    cfg = T.TierConfig(hbm_budget_bytes=lf * 2 * d * 2, d_k=d, d_v=d, block_size=B)
    rng = np.random.default_rng(1)
    pk = O.fp16_round(rng.standard_normal((2, 300, d)))
    pv = O.fp16_round(rng.standard_normal((2, 300, d)))
    src = T.MultiStreamEngine(cfg, n_streams=2)
    src.prefill(pk, pv)
    p0, p1 = tmp_path / "a", tmp_path / "b"
    src.dump_slow_tier(0, p0)
    src.dump_slow_tier(1, p1)
    good = p0.read_bytes()

    def fresh(c=cfg):
        return T.MultiStreamEngine(c, n_streams=2)

    with pytest.raises(T.ShapeError):  # one file per stream
        fresh().restore_slow_tier([p0])
    bad = tmp_path / "bad"
    bad.write_bytes(b"XXKVTIER" + good[8:])
    with pytest.raises(T.IntegrityError, match="bad magic"):
        fresh().restore_slow_tier([bad, p1])
    bad.write_bytes(good[:-5])
    with pytest.raises(T.IntegrityError, match="truncated"):
        fresh().restore_slow_tier([p0, bad])
    bad.write_bytes(good + b"\0")
    with pytest.raises(T.IntegrityError, match="trailing"):
        fresh().restore_slow_tier([p0, bad])
    short = T.MultiStreamEngine(cfg, n_streams=1)
    short.prefill(pk[:1, :200], pv[:1, :200])
    short.dump_slow_tier(0, bad)
    with pytest.raises(T.ShapeError):  # streams must stay in lockstep
        fresh().restore_slow_tier([p0, bad])
    other = T.TierConfig(hbm_budget_bytes=lf * 2 * d * 2, d_k=d, d_v=d, block_size=B,
                         key_bits=4, value_bits=4)
    with pytest.raises(T.ConfigError):
        fresh(other).restore_slow_tier([p0, p1])
    used = fresh()
    used.prefill(pk[:, :10], pv[:, :10])
    with pytest.raises(T.SequencingError):
        used.restore_slow_tier([p0, p1])
    with pytest.raises(T.IoError):
        fresh().restore_slow_tier([p0, tmp_path / "missing"])
    src.close()


def test_restore_wide_key_scales_hbm_tier(gpu, tmp_path):
    # A dump from an fp32 engine can carry key scales no fp16 ring produces
    # (|s| > kTcKeyScaleBound, ttkv_launch.h); restored into an HBM-tier
    # handle at the tensor-core shape, the engine must stay exact (it moves to
    # the CUDA-core slow kernel instead of overflowing the fp16 q * s split).
    T = gpu
    S, d, B, lf, ctx, steps = 2, 128, 128, 512, 1500, 3
    rng = np.random.default_rng(5)
    pk = (rng.standard_normal((S, ctx, d)) * 3e4).astype(np.float32)  # fp32 range
    pv = O.fp16_round(rng.standard_normal((S, ctx, d)))
    refs, paths = [], []
    for s in range(S):
        r = O.RefEngine(lf * 2 * d * 2, d, d, B)
        r.prefill(pk[s], pv[s])
        refs.append(r)
        p = tmp_path / f"w{s}.ttkvtier"
        p.write_bytes(tier_file([r.serialize_block(b) for b in range(r.slow_blocks())]))
        paths.append(p)
    n = refs[0].slow_blocks()
    cfg = T.TierConfig(hbm_budget_bytes=lf * 2 * d * 2, d_k=d, d_v=d, block_size=B)
    eng = T.MultiStreamEngine(cfg, n_streams=S, slow_tier=1)
    eng.restore_slow_tier(paths)
    tail_k = O.fp16_round(pk[:, n * B:] / 3e4)  # the fast tier resumes at fp16 scale
    eng.append(tail_k, pv[:, n * B:])
    for s in range(S):
        refs[s] = O.RefEngine(lf * 2 * d * 2, d, d, B)
        refs[s].prefill(np.concatenate([pk[s, :n * B], tail_k[s]]), pv[s])
    for t in range(steps):
        q = rng.standard_normal((S, 1, d)).astype(np.float32)
        kn = O.fp16_round(rng.standard_normal((S, d)))
        vn = O.fp16_round(rng.standard_normal((S, d)))
        rep = eng.decode_step(q, kn, vn, fetched=True)
        for s in range(S):
            o = refs[s].decode_step(q[s, 0], kn[s], vn[s])
            assert np.array_equal(rep.fetched_blocks[s][0], o["fetched"]), (t, s)
            assert np.all(np.isfinite(rep.output[s, 0]))
            assert rel_err(rep.output[s, 0], o["output"]) < 1e-3
    eng.close()
