"""Quick first-look timing of the decode step (not the bench contract)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2604_19769_b200 as T

def run(name, S, G, ctx, steps=6, copy_mode=0):
    cfg = T.TierConfig(hbm_budget_bytes=4096 * 256 * 2, d_k=128, d_v=128, block_size=128)
    t0 = time.time()
    eng = T.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, reserve_tokens=ctx + 512,
                              copy_mode=copy_mode)
    eng.prefill_synthetic(ctx, seed=1)
    tp = time.time() - t0
    rng = np.random.default_rng(0)
    q = rng.standard_normal((S, G, 128)).astype(np.float32)
    kn = rng.standard_normal((S, 128)).astype(np.float16)
    vn = rng.standard_normal((S, 128)).astype(np.float16)
    eng.decode_step(q, kn, vn)
    eng.set_timing(True)
    eng.kernel_times(reset=True)
    ts = []
    for i in range(steps):
        a = time.time(); r = eng.decode_step(q, kn, vn); ts.append(time.time() - a)
    kt = eng.kernel_times(reset=True)
    print(name, f"copy_mode={copy_mode} prefill {tp:.2f}s step wall ms {np.median(ts)*1e3:.2f}",
          f"union {r.union_blocks} pcie {r.pcie_bytes/1e9:.3f} GB -> {r.pcie_bytes/np.median(ts)/1e9:.1f} GB/s",
          {k: round(v / steps, 3) for k, v in kt.items() if k.startswith('ms_')}, flush=True)
    eng.close()

if __name__ == "__main__":
    run("cfg1", 32, 1, 32768)
    run("cfg1", 32, 1, 32768, copy_mode=2)
    run("cfg2", 256, 4, 131072, steps=4)
    run("cfg2", 256, 4, 131072, steps=4, copy_mode=2)
