"""Table-6 ablation of the paper as real B200 measurements at cfg2 scale.

The reference emulates the ablation with an analytic simulator
(harness.cpp:56-86, run_ablation 210-221; Table 6).  Here every
variant runs on the B200 engine over the cfg2 shape (LLaMA-3-8B GQA, 32
layers x 8 KV heads x 4 query heads, 128K context, synthetic KV) and the
decode step is timed on the device:
  ttkv              K8/V4, fetch 0.45 per query head, pipelined streaming
  no_pipeline       same selection, serial schedule (bulk PCIe gather, then compute)
  uniform_quant_8_8 K8/V8
  single_tier       fast tier = one block, fetch everything
  fp16_full_fetch   16/16 records (fp16 payloads), fetch everything, serial
Prints one JSON line per method.
  python tools/ablation_b200.py [--ctx N] [--steps K] [--methods a,b]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ctx", type=int, default=131072)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--streams", type=int, default=256)
    ap.add_argument("--heads", type=int, default=4)
    ap.add_argument("--methods", default="ttkv,no_pipeline,uniform_quant_8_8,single_tier,"
                                         "fp16_full_fetch")
    args = ap.parse_args()
    import torch
    import paper_2604_19769_b200 as T
    from paper_2604_19769_b200.harness import effective

    D, B = 128, 128
    base = T.TierConfig(hbm_budget_bytes=4096 * 2 * D * 2, d_k=D, d_v=D, block_size=B)
    pol = T.SelectionPolicy(None, 0.45)
    S, G = args.streams, args.heads
    dev = torch.device("cuda", 0)
    for method in args.methods.split(","):
        tier, p, serial = effective(base, pol, method)
        eng = T.MultiStreamEngine(tier, p, n_streams=S, heads_per_stream=G,
                                  reserve_tokens=args.ctx + args.warmup + args.steps + B,
                                  ring_bytes=2, serial_schedule=serial)
        stream = torch.cuda.Stream(device=dev)
        torch.cuda.set_stream(stream)
        eng.set_stream(stream.cuda_stream)
        t0 = time.time()
        eng.prefill_synthetic(args.ctx, seed=7)
        prefill_s = time.time() - t0
        g = torch.Generator(device=dev).manual_seed(0)
        q = torch.randn(S, G, D, device=dev, generator=g)
        k = torch.randn(S, D, device=dev, generator=g).half()
        v = torch.randn(S, D, device=dev, generator=g).half()
        out = torch.empty(S, G, D, device=dev, dtype=torch.float64)
        for _ in range(args.warmup):
            eng.decode_step_device(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), 1)
        torch.cuda.synchronize()
        eng.set_timing(True)
        eng.kernel_times(reset=True)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(args.steps):
            eng.decode_step_device(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), 1)
        b.record()
        torch.cuda.synchronize()
        kt = eng.kernel_times(reset=True)
        union, pcie = eng.step_counters()
        st = eng.state()
        ms = a.elapsed_time(b) / args.steps
        print(json.dumps({
            "method": method, "ctx": args.ctx, "streams": S, "heads": G,
            "key_bits": tier.key_bits, "value_bits": tier.value_bits,
            "fetch_fraction": p.fetch_fraction, "serial": serial, "l_fast": st["l_fast"],
            "ms_per_step": ms, "tok_per_s": 1000.0 / ms,
            "pcie_gb_per_step": pcie / 1e9, "pcie_gbs": pcie / (ms * 1e-3) / 1e9,
            "modeled_h2g_bytes_per_head": st["modeled_block_bytes"],
            "union_blocks": union, "prefill_s": round(prefill_s, 2),
            "kernel_ms_per_step": {k2[3:]: v2 / args.steps for k2, v2 in kt.items()
                                   if k2.startswith("ms_") and v2 > 0},
        }), flush=True)
        eng.close()
        del eng
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
