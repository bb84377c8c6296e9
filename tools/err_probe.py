"""Worst output relative error vs the oracle at the hot-path shape
(d = B = 128, K8/V4), per slow-tier placement (GPU; not a test)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path[:0] = [ROOT, os.path.join(ROOT, "tests")]
import paper_2604_19769_b200 as T  # noqa: E402
import test_gpu_parity as P  # noqa: E402

for G in (1, 4, 8):
    for st in (0, 1):
        w = P.run_parity(T, S=3, G=G, d=128, B=128, l_fast=512, ctx=5000, steps=4, slow_tier=st)
        print(f"G={G} slow_tier={st} worst rel err {w:.3e}", flush=True)
