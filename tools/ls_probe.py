"""Layer-sequential probe: host issue time vs device time per token (not the
bench contract).  python tools/ls_probe.py [slow_tier] [tokens]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_19769_b200 as T  # noqa: E402


def main():
    slow_tier = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    ntok = int(sys.argv[2]) if len(sys.argv) > 2 else 50
    Lyr, S, G, D, ctx = 32, 8, 4, 128, 131072
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    cfg = T.TierConfig(hbm_budget_bytes=4096 * 2 * D * 2, d_k=D, d_v=D, block_size=128)
    engs = []
    for layer in range(Lyr):
        e = T.MultiStreamEngine(cfg, T.SelectionPolicy(None, 0.45), n_streams=S, heads_per_stream=G,
                                device=0, reserve_tokens=ctx + 4 * ntok + 512, slow_tier=slow_tier)
        e.set_stream(stream.cuda_stream)
        e.prefill_synthetic(ctx, seed=7000 + layer)
        engs.append(e)
    qs = [torch.randn(S, G, D, device=dev) for _ in range(Lyr)]
    ks = [torch.randn(S, D, device=dev).half() for _ in range(Lyr)]
    vs = [torch.randn(S, D, device=dev).half() for _ in range(Lyr)]
    outs = [torch.empty(S, G, D, device=dev, dtype=torch.float64) for _ in range(Lyr)]

    def token():
        for layer, e in enumerate(engs):
            e.decode_step_device(qs[layer].data_ptr(), ks[layer].data_ptr(), vs[layer].data_ptr(),
                                 outs[layer].data_ptr(), dtype=1)
    for _ in range(5):
        token()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    for _ in range(ntok):
        token()
    t1 = time.perf_counter()
    e1.record()
    torch.cuda.synchronize()
    gpu = e0.elapsed_time(e1) / ntok
    print(f"slow_tier={slow_tier} per token: host issue {1e3 * (t1 - t0) / ntok:.3f} ms, "
          f"device {gpu:.3f} ms ({1e3 * gpu / Lyr:.1f} us/layer)", flush=True)
    # device-only: one token's calls enqueued behind a 50 ms spin, so the host is far ahead
    torch.cuda._sleep(int(1.9e9 * 0.2))
    e0.record()
    for _ in range(3):
        token()
    e1.record()
    torch.cuda.synchronize()
    print(f"  host-ahead device time {e0.elapsed_time(e1) / 3:.3f} ms/token", flush=True)
    for e in engs:
        e.close()


if __name__ == "__main__":
    main()
