"""Programmatic dependent launch changes only WHEN kernels start, never what
they compute: the same decode steps with TTKV_PDL=1 and TTKV_PDL=0 (read once
per process, so each runs in a subprocess) give bit-identical outputs and
selections, on both slow-tier placements."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
import numpy as np
sys.path.insert(0, {root!r})
import paper_2604_19769_b200 as T
S, G, d, ctx = 6, 4, 128, 9000
cfg = T.TierConfig(hbm_budget_bytes=1024 * 2 * d * 2, d_k=d, d_v=d, block_size=128)
eng = T.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, slow_tier={tier})
eng.prefill_synthetic(ctx, seed=3)
rng = np.random.default_rng(11)
outs, fetched = [], []
for t in range(140):  # crosses an eviction
    q = rng.standard_normal((S, G, d)).astype(np.float32)
    k = rng.standard_normal((S, d)).astype(np.float16)
    v = rng.standard_normal((S, d)).astype(np.float16)
    r = eng.decode_step(q, k, v, fetched=(t % 20 == 0))
    outs.append(r.output)
    if t % 20 == 0:
        fetched.append(np.concatenate([np.concatenate(f) for f in r.fetched_blocks]))
np.savez({out!r}, out=np.stack(outs), fetched=np.concatenate(fetched))
"""


@pytest.mark.parametrize("tier", [0, 1])
def test_pdl_on_off_bit_identical(tmp_path, tier):
    res = {}
    for pdl in ("1", "0"):
        out = str(tmp_path / f"pdl{pdl}.npz")
        env = dict(os.environ, TTKV_PDL=pdl)
        subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, tier=tier, out=out)],
                       env=env, check=True, timeout=600)
        res[pdl] = np.load(out)
    assert np.array_equal(res["1"]["out"], res["0"]["out"])
    assert np.array_equal(res["1"]["fetched"], res["0"]["fetched"])
