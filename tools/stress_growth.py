"""Sustained-generation stress (BASELINE configs[4]): cfg2 shape, prefill
128K, then N consecutive decode steps on the device path (default 4096 = 32
fast-tier evictions + quantize-to-DRAM of all 256 streams), every step timed
with CUDA events.  Reports the step-time distribution, eviction steps vs the
rest, drift across the run and the PCIe rate at the end.
  python tools/stress_growth.py [steps] > profiles/r1_stress_growth.json"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2604_19769_b200 as T  # noqa: E402


def main():
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
    S, G, D, B, ctx = 256, 4, 128, 128, 131072
    dev = torch.device("cuda", 0)
    cfg = T.TierConfig(hbm_budget_bytes=4096 * 2 * D * 2, d_k=D, d_v=D, block_size=B)
    eng = T.MultiStreamEngine(cfg, n_streams=S, heads_per_stream=G,
                              reserve_tokens=ctx + steps + 2 * B)
    st = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(st)
    eng.set_stream(st.cuda_stream)
    eng.prefill_synthetic(ctx, seed=99)
    cap0 = eng.state()["block_capacity"]
    gen = torch.Generator(device=dev).manual_seed(0)
    NP = 8
    qs = [torch.randn(S, G, D, device=dev, generator=gen) for _ in range(NP)]
    ks = [torch.randn(S, D, device=dev, generator=gen).half() for _ in range(NP)]
    vs = [torch.randn(S, D, device=dev, generator=gen).half() for _ in range(NP)]
    out = torch.empty(S, G, D, device=dev, dtype=torch.float64)
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    evicted = []
    torch.cuda.synchronize()
    evs[0].record()
    for i in range(steps):
        r = eng.decode_step_device(qs[i % NP].data_ptr(), ks[i % NP].data_ptr(),
                                   vs[i % NP].data_ptr(), out.data_ptr(), dtype=1)
        evs[i + 1].record()
        evicted.append(bool(r.eviction_occurred))
    torch.cuda.synchronize()
    ms = np.array([evs[i].elapsed_time(evs[i + 1]) for i in range(steps)])
    ev = np.array(evicted)
    union, pcie = eng.step_counters()
    stt = eng.state()
    win = min(512, steps // 4)
    res = {
        "workload": "cfg2 shape (256 streams x 4 heads, d=128, K8/V4, 0.45 per head), prefill "
                    f"128K then {steps} consecutive decode steps, slow tier in pinned DRAM",
        "steps": steps, "evictions": int(ev.sum()),
        "slow_blocks_start_end": [stt["slow_blocks"] - int(ev.sum()), stt["slow_blocks"]],
        "arena_reallocations": int(stt["block_capacity"] != cap0),
        "ms_per_step": {"mean": float(ms.mean()), "p50": float(np.percentile(ms, 50)),
                        "p99": float(np.percentile(ms, 99)), "max": float(ms.max()),
                        "min": float(ms.min())},
        "eviction_steps_ms_mean": float(ms[ev].mean()) if ev.any() else None,
        "other_steps_ms_mean": float(ms[~ev].mean()),
        "first_window_ms_mean": float(ms[:win].mean()),
        "last_window_ms_mean": float(ms[-win:].mean()),
        "tokens_per_s": float(1000.0 / ms.mean()),
        "last_step_pcie_gbs": pcie / (ms[-1] * 1e-3) / 1e9,
        "union_blocks_last_step": union,
    }
    eng.close()
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
