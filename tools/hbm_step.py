"""Decode steps with the slow tier resident in HBM (slow_tier=1), for ncu
captures and quick A/B timing of the attention kernels (not the bench
contract).  python tools/hbm_step.py [S] [ctx] [steps] [G]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2604_19769_b200 as T  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
    steps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
    G = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    slow_tier = int(os.environ.get("TTKV_SLOW_TIER", "1"))
    cfg = T.TierConfig(hbm_budget_bytes=4096 * 256 * 2, d_k=128, d_v=128, block_size=128)
    eng = T.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G, reserve_tokens=ctx + 512,
                              slow_tier=slow_tier)
    eng.prefill_synthetic(ctx, seed=1)
    rng = np.random.default_rng(0)
    q = rng.standard_normal((S, G, 128)).astype(np.float32)
    kn = rng.standard_normal((S, 128)).astype(np.float16)
    vn = rng.standard_normal((S, 128)).astype(np.float16)
    eng.decode_step(q, kn, vn)
    eng.set_timing(True)
    eng.kernel_times(reset=True)
    for _ in range(steps):
        r = eng.decode_step(q, kn, vn)
    kt = eng.kernel_times(reset=True)
    st = eng.state()
    slow = kt["ms_slow"] / max(1, kt["n_slow"])
    fast = kt["ms_fast"] / max(1, kt["n_fast"])
    step = kt["ms_step"] / max(1, kt["n_step"])
    gb = r.union_blocks * st["record_bytes"] / 1e9
    print(f"S={S} G={G} ctx={ctx} union={r.union_blocks} step {step:.3f} ms slow {slow:.3f} ms "
          f"({gb / slow * 1e3:.0f} GB/s of records) fast {fast:.3f} ms", flush=True)
    print("   per-kernel ms:", {k[3:]: round(v / max(1, kt["n" + k[2:]]), 4)
                               for k, v in kt.items() if k.startswith("ms_")}, flush=True)
    eng.close()


if __name__ == "__main__":
    main()
