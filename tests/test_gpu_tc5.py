"""The opt-in tcgen05 slow-tier kernel (slow_attn_tc5_kernel, TTKV_SLOW_TC5=1:
tcgen05.mma.kind::i8 on the raw u8 K codes and expanded V codes, TMEM
accumulators) against the CPU oracle, through the same run_parity checks as
the default tensor-core kernel: every head's selection, records bit-exact,
outputs within 1e-3 -- for G = 1..8, group-shared selection, the literal
merge, extreme magnitudes and a long fast tier.  The variable is read once per
process, so the cases run in one subprocess."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

SCRIPT = r"""
import sys
sys.path.insert(0, {root!r})
sys.path.insert(0, {tests!r})
import paper_2604_19769_b200 as T
import test_gpu_parity as P
worst = 0.0
for G, mode, literal in [(1, 0, False), (2, 0, False), (3, 0, False), (4, 0, False),
                         (4, 1, False), (5, 1, False), (8, 0, False), (4, 0, True)]:
    worst = max(worst, P.run_parity(T, S=3, G=G, d=128, B=128, l_fast=512, ctx=5000, steps=4,
                                    mode=mode, literal=literal, slow_tier=1, record_stream=1))
for q_mul, kv_mul in [(3e4, 1.0), (1.0, 2e3), (1e-6, 1e-3), (1e7, 1.0), (3e3, 5e3)]:
    worst = max(worst, P.run_parity(T, S=2, G=4, d=128, B=128, l_fast=512, ctx=3000, steps=3,
                                    slow_tier=1, q_mul=q_mul, kv_mul=kv_mul, record_stream=1))
P.run_parity(T, S=4, G=4, d=128, B=128, l_fast=16384, ctx=16384 + 200, steps=4, slow_tier=1,
             check_blocks=False, record_stream=1)
print("tc5 ok worst", worst)
"""


def test_tcgen05_slow_kernel_parity():
    env = dict(os.environ, TTKV_SLOW_TC5="1")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT,
                                                           tests=os.path.join(ROOT, "tests"))],
                       env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert "tc5 ok" in r.stdout
