"""Launch modes change only WHEN kernels start, never what they compute: the
same decode steps with programmatic dependent launch on/off (TTKV_PDL) and with
the step replayed as a CUDA graph or launched kernel by kernel (TTKV_GRAPH)
give bit-identical outputs and selections on both slow-tier placements.  The
variables are read once per process, so each mode runs in a subprocess.  The
sequence crosses evictions (graph recapture) and interleaves a host-side
append (the device step position is resynchronized)."""
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
eng = T.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, slow_tier={tier},
                          record_stream={rs})
eng.prefill_synthetic(ctx, seed=3)
rng = np.random.default_rng(11)
outs, fetched = [], []
for t in range(300):  # crosses two evictions
    q = rng.standard_normal((S, G, d)).astype(np.float32)
    k = rng.standard_normal((S, d)).astype(np.float16)
    v = rng.standard_normal((S, d)).astype(np.float16)
    if t == 150:  # a host-side append between decode steps
        eng.append(rng.standard_normal((S, 1, d)).astype(np.float16),
                   rng.standard_normal((S, 1, d)).astype(np.float16))
    r = eng.decode_step(q, k, v, fetched=(t % 20 == 0))
    outs.append(r.output)
    if t % 20 == 0:
        fetched.append(np.concatenate([np.concatenate(f) for f in r.fetched_blocks]))
st = eng.state()
np.savez({out!r}, out=np.stack(outs), fetched=np.concatenate(fetched),
         replays=st["graph_replays"], captures=st["graph_captures"], spec=st["spec_steps"])
"""


# slow tier in pinned DRAM; in HBM with the union record stream; in HBM with
# the speculative stream of every record (slow_attn_tc_spec_kernel)
MODES = [(0, 0), (1, 1), (1, 2)]


def run_mode(tmp_path, mode, **env_over):
    tier, rs = mode
    tag = "_".join(f"{k}{v if v is not None else 'unset'}" for k, v in sorted(env_over.items()))
    out = str(tmp_path / f"{tag}_{tier}_{rs}.npz")
    env = dict(os.environ)
    for k, v in env_over.items():  # None: unset (the library's default)
        if v is None:
            env.pop(k, None)
        else:
            env[k] = v
    subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, tier=tier, rs=rs, out=out)],
                   env=env, check=True, timeout=600)
    r = np.load(out)
    assert int(r["spec"]) == (300 if rs == 2 else 0)  # every step streams speculatively
    return r


@pytest.mark.parametrize("mode", MODES)
def test_pdl_on_off_bit_identical(tmp_path, mode):
    a = run_mode(tmp_path, mode, TTKV_PDL="1")
    b = run_mode(tmp_path, mode, TTKV_PDL="0")
    assert np.array_equal(a["out"], b["out"])
    assert np.array_equal(a["fetched"], b["fetched"])


@pytest.mark.parametrize("mode", MODES)
def test_graph_replay_bit_identical(tmp_path, mode):
    a = run_mode(tmp_path, mode, TTKV_GRAPH="1")
    b = run_mode(tmp_path, mode, TTKV_GRAPH="0")
    # the graph run really replayed: one capture per eviction period (plus
    # the one after the host append), every other non-evicting step a replay
    assert int(a["replays"]) >= 250 and 3 <= int(a["captures"]) <= 6
    assert int(b["replays"]) == 0
    assert np.array_equal(a["out"], b["out"])
    assert np.array_equal(a["fetched"], b["fetched"])


@pytest.mark.parametrize("mode", MODES)
def test_host_buffer_steps_replay_by_default(tmp_path, mode):
    """Without TTKV_GRAPH the synchronous host-buffer call replays its step as
    a graph (it waits for every step, so no cross-step overlap is lost)."""
    a = run_mode(tmp_path, mode, TTKV_GRAPH=None)
    b = run_mode(tmp_path, mode, TTKV_GRAPH="0")
    assert int(a["replays"]) >= 250 and int(b["replays"]) == 0
    assert np.array_equal(a["out"], b["out"])
    assert np.array_equal(a["fetched"], b["fetched"])


@pytest.mark.parametrize("graph", ["0", "1"])
def test_device_join_bit_identical(tmp_path, graph):
    """The combine joining the fast tier on the device (TTKV_DEV_JOIN=1: an
    epoch counter the fast tier's last CTA advances, no event wait on the
    record stream) gives the same bits as the event join, launched directly
    and replayed as a graph, across evictions and a host-side append."""
    mode = (1, 1)  # HBM tier, union stream: the fused selection forks the fast tier early
    a = run_mode(tmp_path, mode, TTKV_DEV_JOIN="1", TTKV_GRAPH=graph)
    b = run_mode(tmp_path, mode, TTKV_DEV_JOIN="0", TTKV_GRAPH=graph)
    assert np.array_equal(a["out"], b["out"])
    assert np.array_equal(a["fetched"], b["fetched"])
