"""Prefill (bulk append + batched evict_quantize) timing at cfg2 scale.
  python tools/prefill_time.py [S] [ctx] [slow_tier]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2604_19769_b200 as T  # noqa: E402

S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
tier = int(sys.argv[3]) if len(sys.argv) > 3 else 0
cfg = T.TierConfig(hbm_budget_bytes=4096 * 256 * 2, d_k=128, d_v=128, block_size=128)
eng = T.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=4, reserve_tokens=ctx + 512,
                          slow_tier=tier)
eng.prefill_synthetic(4096, seed=1)  # warm-up: kernels loaded, staging sized
eng.synchronize()
eng.close()
eng = T.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=4, reserve_tokens=ctx + 512,
                          slow_tier=tier)
eng.set_timing(True)
eng.kernel_times(reset=True)
t0 = time.perf_counter()
eng.prefill_synthetic(ctx, seed=1)
eng.synchronize()
wall = time.perf_counter() - t0
kt = eng.kernel_times(reset=True)
st = eng.state()
nrec = S * st["slow_blocks"]
rec_gb = nrec * st["record_bytes"] / 1e9
print(f"S={S} ctx={ctx} tier={'host' if tier == 0 else 'hbm'} wall {wall * 1e3:.1f} ms, "
      f"evict {kt['ms_evict']:.1f} ms over {kt['n_evict']} launches -> "
      f"{rec_gb / (kt['ms_evict'] * 1e-3):.1f} GB/s of records ({nrec} records), "
      f"append {kt['ms_append']:.1f} ms", flush=True)
eng.close()
