"""Kernel timeline of layer-sequential decode (torch.profiler / CUPTI): one
token's per-layer kernel start/end on the device, to see what bounds a layer
(not the bench contract).  python tools/ls_trace.py [slow_tier] [S]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_19769_b200 as T  # noqa: E402


def main():
    slow_tier = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    S = int(sys.argv[2]) if len(sys.argv) > 2 else 8
    Lyr, G, D, ctx = 8, 4, 128, 131072
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    cfg = T.TierConfig(hbm_budget_bytes=4096 * 2 * D * 2, d_k=D, d_v=D, block_size=128)
    engs = []
    for layer in range(Lyr):
        e = T.MultiStreamEngine(cfg, T.SelectionPolicy(None, 0.45), n_streams=S, heads_per_stream=G,
                                device=0, reserve_tokens=ctx + 512, slow_tier=slow_tier)
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
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        torch.cuda._sleep(int(1.9e9 * 0.05))  # the host runs ahead: a device-bound timeline
        for _ in range(2):
            token()
        torch.cuda.synchronize()
    path = "/tmp/ls_trace.json"
    prof.export_chrome_trace(path)
    ev = [e for e in json.load(open(path))["traceEvents"]
          if e.get("cat") == "kernel" and "sleep" not in e.get("name", "")]
    ev.sort(key=lambda e: e["ts"])
    t0 = ev[0]["ts"]
    short = lambda n: n.split("(")[0].replace("void ", "").replace("ttkv_dev::", "")[:34]
    last = len(ev) - 1
    for e in ev[-8 * 7:]:
        print(f"{e['ts'] - t0:9.2f} {e['ts'] + e['dur'] - t0:9.2f} dur {e['dur']:7.2f} "
              f"s{e['args'].get('stream', '?'):>3} {short(e['name'])}")
    span = (ev[last]["ts"] + ev[last]["dur"] - ev[len(ev) // 2]["ts"]) / (len(ev) - len(ev) // 2)
    print(f"kernels {len(ev)}; mean per-kernel span {span:.2f} us")


if __name__ == "__main__":
    main()
