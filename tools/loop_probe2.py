"""Per-step device time of back-to-back decode steps under different step
separations (none, an event between steps, per-kernel timing events, a host
synchronize per step) -- not the bench contract.
python tools/loop_probe2.py [S] [ctx] [tier] [G] [steps]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_19769_b200 as T  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
    tier = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    G = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 100
    D = 128
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    cfg = T.TierConfig(hbm_budget_bytes=4096 * 2 * D * 2, d_k=D, d_v=D, block_size=128)
    e = T.MultiStreamEngine(cfg, T.SelectionPolicy(None, 0.45), n_streams=S, heads_per_stream=G,
                            device=0, reserve_tokens=ctx + 8 * steps + 512, slow_tier=tier)
    e.set_stream(stream.cuda_stream)
    e.prefill_synthetic(ctx, seed=5)
    q = torch.randn(S, G, D, device=dev)
    k = torch.randn(S, D, device=dev).half()
    v = torch.randn(S, D, device=dev).half()
    out = torch.empty(S, G, D, device=dev, dtype=torch.float64)

    def step():
        e.decode_step_device(q.data_ptr(), k.data_ptr(), v.data_ptr(), out.data_ptr(), dtype=1)

    def plain():
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record()
        for _ in range(steps):
            step()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / steps

    def per_step_events():
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        torch.cuda.synchronize()
        evs[0].record()
        for i in range(steps):
            step()
            evs[i + 1].record()
        torch.cuda.synchronize()
        d = sorted(evs[i].elapsed_time(evs[i + 1]) for i in range(steps))
        return d[len(d) // 2], evs[0].elapsed_time(evs[-1]) / steps

    def synced():
        d = []
        for _ in range(steps):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            a.record()
            step()
            b.record()
            torch.cuda.synchronize()
            d.append(a.elapsed_time(b))
        d.sort()
        return d[len(d) // 2]

    def timed():
        e.set_timing(True)
        e.kernel_times(reset=True)
        r = plain()
        kt = e.kernel_times(reset=True)
        e.set_timing(False)
        return r, {k2[3:]: round(v2 / max(1, kt["n" + k2[2:]]), 4) for k2, v2 in kt.items()
                   if k2.startswith("ms_")}

    plain()
    print("plain              %.4f ms/step" % plain(), flush=True)
    from torch.profiler import ProfilerActivity, profile
    with profile(activities=[ProfilerActivity.CUDA]):
        r = plain()
    print("plain under CUPTI  %.4f ms/step" % r, flush=True)
    with profile(activities=[ProfilerActivity.CPU]):
        r = plain()
    print("plain, CPU profile %.4f ms/step" % r, flush=True)
    print("event per step     median %.4f, mean %.4f ms/step" % per_step_events(), flush=True)
    print("synced per step    median %.4f ms" % synced(), flush=True)
    r, kt = timed()
    print("kernel events      %.4f ms/step %s" % (r, kt), flush=True)
    print("plain              %.4f ms/step" % plain(), flush=True)
    e.close()


if __name__ == "__main__":
    main()
