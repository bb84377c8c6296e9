"""Small GPU parity cases for compute-sanitizer runs (memcheck / racecheck /
synccheck).  Exercises every kernel family once with tiny shapes."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import paper_2604_19769_b200 as T
import test_gpu_parity as P

cases = [
    dict(S=1, G=1, d=16, B=32, l_fast=128, ctx=300, steps=3),                 # generic CUDA-core
    dict(S=2, G=3, d=20, dv=7, B=24, l_fast=96, ctx=200, steps=3, kb=6, vb=3),  # ragged dims
    dict(S=1, G=4, d=128, B=128, l_fast=256, ctx=700, steps=2),               # TC fast, host slow
    dict(S=1, G=4, d=128, B=128, l_fast=256, ctx=700, steps=2, slow_tier=1),  # TC slow (HBM)
    dict(S=1, G=2, d=64, B=64, l_fast=128, ctx=400, steps=2, literal=True),
    dict(S=1, G=2, d=16, B=32, l_fast=128, ctx=300, steps=2, elem=4),         # fp64 accumulation
    # > 64 slow blocks: the selection sort's cross-warp (stride >= 64) passes
    dict(S=2, G=4, d=128, B=128, l_fast=256, ctx=20000, steps=2, slow_tier=1),
    dict(S=2, G=8, d=32, B=32, l_fast=128, ctx=9000, steps=2),
    # power-of-two q normalization at query magnitudes that overflow fp16
    dict(S=1, G=4, d=128, B=128, l_fast=256, ctx=700, steps=2, slow_tier=1, q_mul=1e7),
    # speculative record stream (every record beside the selection, per-record
    # partials, the compacting combine) and the fused selection cluster kernel
    dict(S=2, G=4, d=128, B=128, l_fast=256, ctx=5000, steps=2, slow_tier=1, record_stream=2),
]
for c in cases:
    P.run_parity(T, **c)
    print("ok", c, flush=True)
