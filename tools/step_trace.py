"""Kernel timeline of back-to-back decode steps of one handle (torch.profiler
/ CUPTI): per-kernel start/end on the device, to see what bounds a step (not
the bench contract).  python tools/step_trace.py [S] [ctx] [slow_tier] [G] [steps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_19769_b200 as T  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
    slow_tier = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    G = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 3
    warm = int(sys.argv[6]) if len(sys.argv) > 6 else 3
    quiet = steps > 8
    D = 128
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    cfg = T.TierConfig(hbm_budget_bytes=4096 * 2 * D * 2, d_k=D, d_v=D, block_size=128)
    e = T.MultiStreamEngine(cfg, T.SelectionPolicy(None, 0.45), n_streams=S, heads_per_stream=G,
                            device=0, reserve_tokens=ctx + 512, slow_tier=slow_tier)
    e.set_stream(stream.cuda_stream)
    e.prefill_synthetic(ctx, seed=5)
    q = torch.randn(S, G, D, device=dev)
    k = torch.randn(S, D, device=dev).half()
    v = torch.randn(S, D, device=dev).half()
    out = torch.empty(S, G, D, device=dev, dtype=torch.float64)

    def step():
        e.decode_step_device(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), dtype=1)
    for _ in range(warm):
        step()
    torch.cuda.synchronize()
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        torch.cuda._sleep(int(1.9e9 * 0.02))  # the host runs ahead: a device-bound timeline
        for _ in range(steps):
            step()
        torch.cuda.synchronize()
    path = "/tmp/step_trace.json"
    prof.export_chrome_trace(path)
    ev = [x for x in json.load(open(path))["traceEvents"]
          if x.get("cat") == "kernel" and "sleep" not in x.get("name", "")]
    ev.sort(key=lambda x: x["ts"])
    t0 = ev[0]["ts"]
    short = lambda n: n.split("(")[0].replace("void ", "").replace("ttkv_dev::", "")[:34]
    for x in (ev[-24:] if quiet else ev):
        print(f"{x['ts'] - t0:9.2f} {x['ts'] + x['dur'] - t0:9.2f} dur {x['dur']:8.2f} "
              f"s{x['args'].get('stream', '?'):>3} {short(x['name'])}")
    slow = [x for x in ev if "slow_attn" in x["name"]]
    fast = [x for x in ev if "fast_attn" in x["name"]]
    if slow and len(slow) == len(fast):
        import statistics as stt
        print("slow dur median %.1f us; fast start - slow start median %.1f us; "
              "fast end - slow end median %.1f us" % (
                  stt.median(x["dur"] for x in slow),
                  stt.median(f["ts"] - s_["ts"] for f, s_ in zip(fast, slow)),
                  stt.median(f["ts"] + f["dur"] - s_["ts"] - s_["dur"] for f, s_ in zip(fast, slow))))
    print(f"kernels {len(ev)}; span {(ev[-1]['ts'] + ev[-1]['dur'] - t0) / steps:.1f} us per step")
    e.close()


if __name__ == "__main__":
    main()
