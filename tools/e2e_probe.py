import time, sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_2604_19769_b200 as T
from paper_2604_19769_b200 import engine as E
S, G, ctx = 256, 4, 131072
cfg = T.TierConfig(hbm_budget_bytes=4096 * 256 * 2, d_k=128, d_v=128, block_size=128)
eng = T.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, reserve_tokens=ctx + 512, slow_tier=1)
eng.prefill_synthetic(ctx, seed=1)
rng = np.random.default_rng(0)
q = rng.standard_normal((S, G, 128)).astype(np.float32)
kn = rng.standard_normal((S, 128)).astype(np.float16)
vn = rng.standard_normal((S, 128)).astype(np.float16)
for _ in range(5): eng.decode_step(q, kn, vn)
n = 30
t0 = time.perf_counter()
for _ in range(n): eng.decode_step(q, kn, vn)
t1 = time.perf_counter()
print("python decode_step ms", (t1 - t0) * 1e3 / n)
import ctypes as C
from paper_2604_19769_b200 import _lib as L
out = np.zeros((S, G, 128), np.float64)
rep = L.StepReportC()
lib = eng._lib
qp, kp, vp, op = (x.ctypes.data_as(C.c_void_p) for x in (q.reshape(-1), kn, vn, out))
t0 = time.perf_counter()
for _ in range(n): lib.ttkv_gpu_decode_step(eng._h, qp, kp, vp, 1, op, C.byref(rep))
t1 = time.perf_counter()
print("raw C decode_step ms (reused out)", (t1 - t0) * 1e3 / n)
t0 = time.perf_counter()
for _ in range(n): o = np.zeros((S, G, 128), np.float64)
t1 = time.perf_counter()
print("np.zeros ms", (t1 - t0) * 1e3 / n)
