"""Back-to-back decode steps timed with CUDA events under variants of the
bench's timed loop (same / rotating inputs, with / without the NVML clock
sampler thread), to find what separates the bench's ms/step from a kernel
timeline (not the bench contract).  python tools/loop_probe.py [S] [ctx] [tier] [G] [steps]"""
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2604_19769_b200 as T  # noqa: E402


def main():
    S = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    ctx = int(sys.argv[2]) if len(sys.argv) > 2 else 131072
    tier = int(sys.argv[3]) if len(sys.argv) > 3 else 1
    G = int(sys.argv[4]) if len(sys.argv) > 4 else 4
    steps = int(sys.argv[5]) if len(sys.argv) > 5 else 400
    D = 128
    dev = torch.device("cuda", 0)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    cfg = T.TierConfig(hbm_budget_bytes=4096 * 2 * D * 2, d_k=D, d_v=D, block_size=128)
    e = T.MultiStreamEngine(cfg, T.SelectionPolicy(None, 0.45), n_streams=S, heads_per_stream=G,
                            device=0, reserve_tokens=ctx + 8 * steps + 512, slow_tier=tier)
    e.set_stream(stream.cuda_stream)
    e.prefill_synthetic(ctx, seed=5)
    gen = torch.Generator(device=dev).manual_seed(0)
    qs = [torch.randn(S, G, D, device=dev, generator=gen) for _ in range(4)]
    ks = [torch.randn(S, D, device=dev, generator=gen).half() for _ in range(4)]
    vs = [torch.randn(S, D, device=dev, generator=gen).half() for _ in range(4)]
    out = torch.empty(S, G, D, device=dev, dtype=torch.float64)

    def run(rot, sampler):
        stop = threading.Event()
        th = None
        if sampler:
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(0)

            def loop():
                while not stop.wait(0.01):
                    pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
            th = threading.Thread(target=loop, daemon=True)
            th.start()
        import time
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record()
        for i in range(steps):
            j = i % 4 if rot else 0
            e.decode_step_device(qs[j].data_ptr(), ks[j].data_ptr(), vs[j].data_ptr(),
                                 out.data_ptr(), dtype=1)
        b.record()
        host = (time.perf_counter() - t0) * 1e3 / steps
        torch.cuda.synchronize()
        stop.set()
        return a.elapsed_time(b) / steps, host

    run(True, False)
    for rot, smp in ((False, False), (True, False), (False, True), (True, True), (False, False)):
        dv, hs = run(rot, smp)
        print(f"rotate={rot} sampler={smp}: {dv:.4f} ms/step (host issue {hs:.4f} ms/step)", flush=True)
    e.close()


if __name__ == "__main__":
    main()
