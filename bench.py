#!/usr/bin/env python
"""Benchmark of the TTKV decode hot path on B200 (BASELINE.json metric).

Default workload (N=1): BASELINE.json configs[1] (cfg2) -- LLaMA-3-8B GQA
decode at 128K context, batch 1, all 32 layers x 8 KV heads = 256 KV streams,
4 query heads each, d=128, 4096-token fp16 fast tier per stream, K8/V4 slow
tier in pinned host DRAM, fetch fraction 0.45, per-query-head selection
(== 1024 reference Engines).  One step = one decode step of every layer/head
(one generated token per request).
N>1 (configs[3], cfg4): the same request head-sharded over N GPUs -- rank r
owns KV heads [8r/N, 8(r+1)/N) of every layer, streams its records over its
own PCIe link, and the combine kernel writes every head's output into every rank over
NVLink peer memory (the all-gather fused into the combine; NCCL as fallback).
--workload cfg1|cfg3|cfg5 selects the other BASELINE configs (cfg3 shards
by request at N>1, no collective).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

`value` is tokens/s with inputs resident in HBM; `e2e` is the same metric
through the public C ABI with host buffers (q/k/v H2D + output D2H inside the
timed region).  `--impl reference` times the unmodified reference engine
(oracle/_ref) on the host cores on a bounded sample, extrapolated.
"""
import argparse
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
try:
    ALL_CPUS = os.sched_getaffinity(0)  # restored for the host-core CPU baseline
except Exception:  # noqa: BLE001
    ALL_CPUS = None

D, B, L_FAST, FRAC = 128, 128, 4096, 0.45
UNIT = "tok/s"
WORKLOADS = {
    "cfg1": dict(layers=1, kv_heads=32, G=1, batch=1, ctx=32768,
                 desc="cfg1: single-layer LLaMA-7B-shape MHA (32 heads, d=128), 32K ctx, batch 1"),
    "cfg2": dict(layers=32, kv_heads=8, G=4, batch=1, ctx=131072,
                 desc="cfg2: LLaMA-3-8B GQA 32L x 8KV x 4Q, 128K ctx, batch 1"),
    "cfg3": dict(layers=32, kv_heads=8, G=4, batch=16, ctx=32768,
                 desc="cfg3: LLaMA-3-8B GQA 32L x 8KV x 4Q, 32K ctx, batch 16"),
    "cfg5": dict(layers=32, kv_heads=8, G=4, batch=1, ctx=262144,
                 desc="cfg5: LLaMA-3-8B GQA at 256K ctx (end of 128K->256K growth)"),
}


def metric_for(w):
    if w == "cfg2":
        return "decode tokens/s at 128K ctx (LLaMA-3-8B GQA, all layers, batch 1)"
    return f"decode tokens/s ({WORKLOADS[w]['desc']})"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=None,
                   help="timed steps (default 10; cfg5: per growth point, default B=128)")
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--workload", default="cfg2", choices=sorted(WORKLOADS))
    p.add_argument("--ctx", type=int, default=None, help="override the workload's context")
    p.add_argument("--group-select", action="store_true",
                   help="one selection per KV head (q' = sum_g q_g) instead of per query head")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--slow-tier", default="host", choices=["host", "device"])
    p.add_argument("--layer-sequential", action="store_true",
                   help="one dependent decode call per layer (one handle per layer)")
    a = p.parse_args()
    a.steps_given = a.steps is not None
    if a.steps is None:
        a.steps = 10
    a.w = dict(WORKLOADS[a.workload])
    if a.ctx:
        a.w["ctx"] = a.ctx
    return a


def dist_env():
    return (int(os.environ.get("RANK", 0)), int(os.environ.get("LOCAL_RANK", 0)),
            int(os.environ.get("WORLD_SIZE", 1)))


# ---------------------------------------------------------------------------
# reference arm / cpu baseline (oracle/_ref: the unmodified reference engine)
# ---------------------------------------------------------------------------
def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def ref_sample(ctx, steps, G, engines=None, threads=None):
    """Runs `engines` reference Engines (one per (stream, query head)) at ctx,
    prefilled, then `steps` decode steps on `threads` host threads.  Returns
    per-step wall ms of the sample."""
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    import numpy as np
    import _oracle as O
    if not O.ref_available():
        raise RuntimeError("oracle/_ref/libttkv_ref.so missing (built by __graft_entry__.build())")
    if ALL_CPUS:
        os.sched_setaffinity(0, ALL_CPUS)
    threads = threads or host_cores()
    engines = engines or threads
    ms = np.zeros(steps, np.float64)
    pre = C.c_double()
    rc = O.ref().ref_bench_decode(engines, G, ctx, steps, threads, L_FAST * 2 * D * 2, D, B, 8, 4,
                                  FRAC, 1234, ms, C.byref(pre))
    if rc != 0:
        raise RuntimeError(O.ref().ref_last_error().decode())
    return ms, pre.value, engines, threads


def scale_note(engines, total):
    return ("all engines, not extrapolated" if engines >= total else
            f"extrapolated x{total / engines:g} to {total} engines")


def cpu_throughput(ms_step, engines, total_engines, tokens_per_step):
    """tokens/s of the full workload, extrapolated linearly from the sample:
    a full step needs total_engines/engines sample steps."""
    full_ms = ms_step * total_engines / engines
    return tokens_per_step * 1000.0 / full_ms


def run_reference(args):
    rank, _, world = dist_env()
    if rank != 0:
        return
    w = args.w
    S = w["layers"] * w["kv_heads"] * w["batch"]
    total_engines = S * w["G"]  # one reference Engine per (stream, q-head)
    n = args.warmup + args.steps
    # small workloads (cfg1: 32 Engines) run in full; larger ones are sampled
    ms, pre_s, engines, threads = ref_sample(w["ctx"], n, w["G"],
                                             engines=total_engines if total_engines <= 64 else None)
    timed = ms[args.warmup:]
    vals = [cpu_throughput(m, engines, total_engines, w["batch"]) for m in timed]
    value = statistics.mean(vals)
    sample = (f"{engines} reference Engines (1 per stream x q-head) at {w['ctx']} ctx on "
              f"{threads} threads, {args.steps} timed decode steps after {args.warmup} warm-up; "
              f"{scale_note(engines, total_engines)}")
    line = {
        "impl": "reference", "metric": metric_for(args.workload), "value": value, "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": w["batch"] * 1000.0 / value, "higher_is_better": True,
        "scaling": "strong" if world > 1 and w["batch"] == 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference GaussianSource)",
        "config": {"workload": w["desc"], "ctx": w["ctx"], "streams": S,
                   "heads_per_stream": w["G"], "d": D, "block": B, "l_fast": L_FAST,
                   "bits": "K8/V4", "fetch_fraction": FRAC},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "reference",
                         "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "sample_ms_per_step": [round(float(x), 2) for x in timed],
        "prefill_s": round(pre_s, 2),
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------
class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.proc = None
        self.lines = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        return self

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [l for l in out.splitlines() if l.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in self.lines:
            f = [x.strip() for x in l.split(",")]
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------
def measure_h2d_peak(torch, dev):
    """pinned H2D copy-engine peak (256 MiB, best of 10): the PCIe roofline."""
    n = 256 << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    best = 1e30
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        d.copy_(h, non_blocking=True)
        b.record()
        b.synchronize()
        best = min(best, a.elapsed_time(b))
    return n / best / 1e6  # GB/s


def load_traffic():
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as f:
            return json.load(f)
    except Exception:
        return None


def bind_numa(device):
    """Pin this rank to the CPUs of its GPU's NUMA node before the pinned
    slow-tier arena is allocated, so cudaHostAlloc's pages land on the node
    whose memory controller sits next to that GPU's PCIe root port (8-GPU
    boxes have two sockets; each rank streams ~51 GB/s from host DRAM)."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(device)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
    except Exception:  # noqa: BLE001 -- affinity is an optimisation only
        pass


def init_dist(torch, dist, local, world):
    """One process per GPU: NCCL over NVLink.  TTKV_DIST_BACKEND=gloo with
    TTKV_SHARE_DEVICE=1 runs every rank on cuda:0 (exercises the N>1 path on a
    1-GPU box; the NVLink numbers need NCCL and one GPU per rank)."""
    share = os.environ.get("TTKV_SHARE_DEVICE") == "1"
    dev = torch.device("cuda", 0 if share else local)
    bind_numa(dev.index)
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("TTKV_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return dev


def allreduce_max(t):
    """max over ranks (device tensor; staged through the host for gloo)."""
    import torch.distributed as dist
    if not dist.is_initialized() or dist.get_world_size() == 1:
        return t
    if dist.get_backend() == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return t
    c = t.cpu()
    dist.all_reduce(c, op=dist.ReduceOp.MAX)
    return c.to(t.device)


def setup_gather(eng, plan):
    """N>1 with heads sharded: the combine kernel writes every rank's rows over
    peer memory (PeerGather, no separate collective); NCCL all_gather if the
    IPC mapping is unavailable or TTKV_GATHER=nccl."""
    if not plan.needs_gather:
        return None, "none"
    if os.environ.get("TTKV_GATHER", "peer") == "peer":
        from paper_2604_19769_b200.sharding import PeerGather
        try:
            return PeerGather(eng, plan), "combine fused with the all-gather over peer memory"
        except Exception as e:  # noqa: BLE001
            print(f"peer gather unavailable ({e}); using NCCL all_gather", file=sys.stderr)
    return None, "NCCL all_gather"


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2604_19769_b200 as T
    from paper_2604_19769_b200.sharding import ShardPlan, gather_outputs

    rank, local, world = dist_env()
    dev = init_dist(torch, dist, local, world)
    w = args.w
    G, ctx, batch = w["G"], w["ctx"], w["batch"]
    mode = "heads" if batch == 1 else "requests"
    plan = ShardPlan(rank, world, w["layers"], w["kv_heads"], batch, mode)
    S = plan.n_local  # streams on this rank

    cfg = T.TierConfig(hbm_budget_bytes=L_FAST * 2 * D * 2, d_k=D, d_v=D, bytes_full_precision=2,
                       block_size=B, key_bits=8, value_bits=4, fetch_fraction=FRAC)
    n_steps_total = args.warmup + 2 * args.steps + 8  # timed + kernel-breakdown + e2e steps
    eng = T.MultiStreamEngine(cfg, T.SelectionPolicy(None, FRAC), n_streams=S,
                              heads_per_stream=G, group_select=args.group_select, device=dev.index,
                              reserve_tokens=ctx + n_steps_total + B,
                              slow_tier=0 if args.slow_tier == "host" else 1)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    t0 = time.time()
    eng.prefill_synthetic(ctx, seed=1000 + rank)
    prefill_s = time.time() - t0
    if world > 1:  # all ranks at once: the concurrent per-GPU link peak
        dist.barrier()
    h2d_peak = measure_h2d_peak(torch, dev)

    gen = torch.Generator(device=dev).manual_seed(rank)
    NPOOL = 4
    qs = [torch.randn(S, G, D, device=dev, generator=gen) for _ in range(NPOOL)]
    ks = [torch.randn(S, D, device=dev, generator=gen).half() for _ in range(NPOOL)]
    vs = [torch.randn(S, D, device=dev, generator=gen).half() for _ in range(NPOOL)]
    out = torch.empty(S, G, D, device=dev, dtype=torch.float64)

    pg, gather_kind = setup_gather(eng, plan)

    def step(i):
        eng.decode_step_device(qs[i % NPOOL].data_ptr(), ks[i % NPOOL].data_ptr(),
                               vs[i % NPOOL].data_ptr(), out.data_ptr(), dtype=1)
        if plan.needs_gather and pg is None:  # per-head outputs -> every rank (NCCL)
            gather_outputs(out, plan)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    for i in range(args.warmup):
        step(i)
    barrier()
    st0 = eng.state()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev.index) as clk:
        barrier()
        ev0.record()
        for i in range(args.steps):
            step(args.warmup + i)
        ev1.record()
        barrier()
    ms_total = ev0.elapsed_time(ev1)
    st1 = eng.state()
    union_last, _ = eng.step_counters()
    launches = st1["launches"] - st0["launches"]
    # per-kernel breakdown (CUDA events around every kernel) on separate steps,
    # so the timed region above carries no per-kernel instrumentation
    n_kt = min(args.steps, 5)
    eng.kernel_times(reset=True)
    eng.set_timing(True)
    for i in range(n_kt):
        step(args.warmup + args.steps + i)
    barrier()
    eng.set_timing(False)
    kt = eng.kernel_times(reset=True)

    # --- e2e through the public C ABI with host buffers -----------------------
    rng = np.random.default_rng(rank)
    hq = [rng.standard_normal((S, G, D)).astype(np.float32) for _ in range(NPOOL)]
    hk = [rng.standard_normal((S, D)).astype(np.float16) for _ in range(NPOOL)]
    hv = [rng.standard_normal((S, D)).astype(np.float16) for _ in range(NPOOL)]
    h2d = hq[0].nbytes + hk[0].nbytes + hv[0].nbytes
    d2h = S * G * D * 8 * (world if plan.needs_gather else 1)
    barrier()
    t_e2e0 = time.perf_counter()
    for i in range(args.steps):
        r = eng.decode_step(hq[i % NPOOL], hk[i % NPOOL], hv[i % NPOOL])
        if pg is not None:
            _ = pg.host()
        elif plan.needs_gather:
            _ = gather_outputs(torch.from_numpy(r.output).to(dev), plan).cpu()
    barrier()
    e2e_ms = (time.perf_counter() - t_e2e0) * 1000.0 / args.steps

    # --- max over ranks ---------------------------------------------------------
    vals = torch.tensor([ms_total, e2e_ms], device=dev, dtype=torch.float64)
    if world > 1:
        vals = allreduce_max(vals)
    ms_total, e2e_ms = float(vals[0]), float(vals[1])
    ms_step = ms_total / args.steps
    tokens_per_step = batch  # one generated token per request per step
    value = tokens_per_step * 1000.0 / ms_step

    # --- roofline of the dominant kernel (slow_stream_attn, PCIe-bound) ---------
    rec = st1["record_bytes"]
    payload = st1["payload_bytes"]  # params are staged from the HBM mirror
    n_slow = kt["n_slow"] or 1
    slow_ms = kt["ms_slow"] / n_slow
    pcie_bytes_launch = union_last * payload
    achieved = pcie_bytes_launch / (slow_ms * 1e-3) / 1e9 if slow_ms > 0 else 0.0
    fast_ms = kt["ms_fast"] / max(1, kt["n_fast"])
    F = st1["fast_tokens"]
    fast_bytes = S * F * 2 * D * 2
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    hbm_bytes_step = fast_bytes + S * st1["slow_blocks"] * D * 4 + union_last * (rec - payload)
    host_tier = args.slow_tier == "host"
    if host_tier:  # records cross PCIe (zero-copy); params + centroids + fast tier from HBM
        t_roof_ms = max(hbm_bytes_step / (hbm_peak * 1e9),
                        pcie_bytes_launch / (h2d_peak * 1e9)) * 1e3
        roof = {"bound": "pcie_h2d", "kernel": "slow_stream_attn", "achieved": achieved,
                "peak": h2d_peak, "unit": "GB/s", "frac": achieved / h2d_peak,
                "peak_source": "pinned cudaMemcpy H2D 256 MiB best of 10, measured in this run" +
                               (", all ranks concurrently" if world > 1 else "")}
    else:  # HBM-resident slow tier: every byte of the step is an HBM byte
        hbm_bytes_step += pcie_bytes_launch
        t_roof_ms = hbm_bytes_step / (hbm_peak * 1e9) * 1e3
        slow_bytes = union_last * rec  # payload from the arena + params from the mirror
        ach = slow_bytes / (slow_ms * 1e-3) / 1e9 if slow_ms > 0 else 0.0
        roof = {"bound": "hbm", "kernel": "slow_attn_tc", "achieved": ach, "peak": hbm_peak,
                "unit": "GB/s", "frac": ach / hbm_peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)"}
        pcie_bytes_launch = 0
    traffic = load_traffic() if args.workload == "cfg2" else None

    line = {
        "metric": metric_for(args.workload), "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 and mode == "heads" else "weak", "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (device N(0,1) KV rounded to fp16, random queries)",
        "config": {
            "workload": w["desc"] + (f", head-sharded over {world} GPUs" if plan.needs_gather else
                                     (f", request-sharded over {world} GPUs" if world > 1 else "")),
            "output_gather": gather_kind,
            "ctx": ctx, "streams_per_gpu": S, "heads_per_stream": G, "batch": batch, "d": D,
            "block": B, "l_fast": L_FAST, "bits": "K8/V4", "fetch_fraction": FRAC,
            "selection": "group-shared" if args.group_select else "per-query-head (reference)",
            "slow_tier": "pinned host DRAM, zero-copy PCIe" if args.slow_tier == "host" else "HBM",
            "storage": "fp16 ring, u8 keys / u4 values, f32 params",
            "parallelism": f"{mode}-shard{world}" if world > 1 else "single",
            "l2": "inputs larger than L2 (fp16 ring + slow tier far above 126 MB)",
        },
        "roofline": {
            **roof,
            "traffic": (traffic.get("slow_dram_bytes_per_launch") if host_tier
                        else traffic.get("slow_tc_hbm_dram_bytes_per_launch")) if traffic else None,
            "pcie_traffic": (traffic.get("slow_sysmem_read_bytes_per_launch")
                             if traffic and host_tier else None),
            "algorithmic_bytes_per_launch": pcie_bytes_launch if host_tier else union_last * rec,
            "launch_ms": slow_ms,
            "tier_roofline_ms": t_roof_ms, "tier_frac": t_roof_ms / ms_step,
            "fast_attn": {"ms": fast_ms, "hbm_gbs": fast_bytes / (fast_ms * 1e-3) / 1e9
                          if fast_ms > 0 else None,
                          "hbm_peak": hbm_peak, "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                          "note": "timed concurrently with slow_stream_attn on a second stream"},
        },
        "pcie_bytes_per_token": pcie_bytes_launch * world / tokens_per_step,
        "union_blocks_per_step": union_last,
        "kernel_ms_per_step": {k[3:]: v / n_kt for k, v in kt.items() if k.startswith("ms_")},
        "gpu_launches": launches,
        "e2e": {"value": tokens_per_step * 1000.0 / e2e_ms, "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms},
        "prefill_s": round(prefill_s, 2),
    }
    if rank == 0:
        line["clocks"] = clk.summary()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            total = S * G
            ms, _, engines, threads = ref_sample(ctx, 2, G,
                                                 engines=total if total <= 64 else None)
            cv = cpu_throughput(float(ms[-1]), engines, total, tokens_per_step)
            line["cpu_baseline"] = {
                "value": cv, "unit": UNIT, "cores": threads, "kind": "reference",
                "sample": (f"{engines} unmodified reference Engines at {ctx} ctx, "
                           f"2 decode steps on {threads} threads (last timed: "
                           f"{ms[-1]:.0f} ms), {scale_note(engines, total)}")}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": host_cores(),
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    eng.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


GROWTH_POINTS = (131072, 163840, 196608, 229376, 262144)


def growth_ms_per_step(curve):
    """Mean ms/step of generating every token between the first and the last
    sampled context: the trapezoid integral of ms/step over the context
    divided by the tokens generated (one point: its own ms/step)."""
    if len(curve) == 1:
        return curve[0]["ms_per_step"]
    xs = [c["ctx_start"] for c in curve]
    ys = [c["ms_per_step"] for c in curve]
    total_ms = sum((xs[i + 1] - xs[i]) * (ys[i] + ys[i + 1]) / 2 for i in range(len(xs) - 1))
    return total_ms / (xs[-1] - xs[0])


def run_growth(args):
    """cfg5 (BASELINE configs[4]): sustained generation 128K -> 256K.

    Generating 131,072 tokens takes hours, so the growth curve is sampled:
    at each context point (prefill/bulk-append to it, W warm-up steps) one
    full eviction period of B=128 consecutive decode steps is timed, so each
    window contains exactly one fast-tier eviction + quantize-to-DRAM of all
    S streams (a B-th of the steps, as in sustained generation).  Step times
    are recorded per step with CUDA events on the engine's stream.  `value` is
    131,072 tokens / the trapezoid integral of ms/step over the growth, i.e.
    the sustained generation rate of the 128K->256K run; `ms_per_step` is its
    reciprocal."""
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2604_19769_b200 as T
    from paper_2604_19769_b200.sharding import ShardPlan, gather_outputs

    rank, local, world = dist_env()
    dev = init_dist(torch, dist, local, world)
    w = args.w
    G = w["G"]
    plan = ShardPlan(rank, world, w["layers"], w["kv_heads"], w["batch"], "heads")
    S = plan.n_local
    K = args.steps if args.steps_given else B
    points = GROWTH_POINTS if not args.ctx else (args.ctx,)
    cfg = T.TierConfig(hbm_budget_bytes=L_FAST * 2 * D * 2, d_k=D, d_v=D, bytes_full_precision=2,
                       block_size=B, key_bits=8, value_bits=4, fetch_fraction=FRAC)
    eng = T.MultiStreamEngine(cfg, T.SelectionPolicy(None, FRAC), n_streams=S,
                              heads_per_stream=G, group_select=args.group_select, device=dev.index,
                              reserve_tokens=points[-1] + len(points) * (args.warmup + K) + 2 * B,
                              slow_tier=0 if args.slow_tier == "host" else 1)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    eng.set_stream(stream.cuda_stream)
    if world > 1:  # all ranks at once: the concurrent per-GPU link peak
        dist.barrier()
    h2d_peak = measure_h2d_peak(torch, dev)
    gen = torch.Generator(device=dev).manual_seed(rank)
    NPOOL = 4
    qs = [torch.randn(S, G, D, device=dev, generator=gen) for _ in range(NPOOL)]
    ks = [torch.randn(S, D, device=dev, generator=gen).half() for _ in range(NPOOL)]
    vs = [torch.randn(S, D, device=dev, generator=gen).half() for _ in range(NPOOL)]
    out = torch.empty(S, G, D, device=dev, dtype=torch.float64)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    pg, gather_kind = setup_gather(eng, plan)
    curve, non_ev, evict_ms, launches, prefill_s = [], [], [], 0, 0.0
    kt_tot = {}
    pcie_last = union_last = 0
    with Clocks(dev.index) as clk:
        for pi, ctx in enumerate(points):
            have = eng.state()["appended"]
            if have < ctx:
                t0 = time.time()
                eng.prefill_synthetic(ctx - have, seed=1000 + 17 * pi + rank)
                torch.cuda.synchronize()
                prefill_s += time.time() - t0
            for i in range(args.warmup):
                eng.decode_step_device(qs[i % NPOOL].data_ptr(), ks[i % NPOOL].data_ptr(),
                                       vs[i % NPOOL].data_ptr(), out.data_ptr(), dtype=1)
            barrier()
            st0 = eng.state()
            eng.kernel_times(reset=True)
            eng.set_timing(True)
            evs = [torch.cuda.Event(enable_timing=True) for _ in range(K + 1)]
            ev_flags = []
            barrier()
            evs[0].record()
            for i in range(K):
                rep = eng.decode_step_device(qs[i % NPOOL].data_ptr(), ks[i % NPOOL].data_ptr(),
                                             vs[i % NPOOL].data_ptr(), out.data_ptr(), dtype=1)
                if plan.needs_gather and pg is None:
                    gather_outputs(out, plan)
                evs[i + 1].record()
                ev_flags.append(bool(rep.eviction_occurred))
            barrier()
            eng.set_timing(False)
            kt = eng.kernel_times(reset=True)
            for k_, v_ in kt.items():
                kt_tot[k_] = kt_tot.get(k_, 0) + v_
            st1 = eng.state()
            launches += st1["launches"] - st0["launches"]
            step_ms = [evs[i].elapsed_time(evs[i + 1]) for i in range(K)]
            tot = torch.tensor([evs[0].elapsed_time(evs[K])], device=dev, dtype=torch.float64)
            if world > 1:
                tot = allreduce_max(tot)
            union_last, pcie_last = eng.step_counters()
            ev_idx = [i for i, f in enumerate(ev_flags) if f]
            evict_ms += [step_ms[i] for i in ev_idx]
            non_ev += [m for i, m in enumerate(step_ms) if not ev_flags[i]]
            curve.append({"ctx_start": st0["appended"], "slow_blocks": st1["slow_blocks"],
                          "ms_per_step": float(tot[0]) / K,
                          "p50_ms": float(np.percentile(step_ms, 50)),
                          "p95_ms": float(np.percentile(step_ms, 95)),
                          "max_ms": float(max(step_ms)),
                          "eviction_steps": len(ev_idx),
                          "eviction_step_ms": [round(step_ms[i], 3) for i in ev_idx],
                          "evict_kernel_ms": kt["ms_evict"] / max(1, kt["n_evict"]),
                          "slow_kernel_ms": kt["ms_slow"] / max(1, kt["n_slow"]),
                          "union_blocks": union_last})

    ms_step = growth_ms_per_step(curve)
    value = 1000.0 / ms_step

    # e2e through the C ABI with host buffers, at the last (256K) point
    rng = np.random.default_rng(rank)
    hq = [rng.standard_normal((S, G, D)).astype(np.float32) for _ in range(NPOOL)]
    hk = [rng.standard_normal((S, D)).astype(np.float16) for _ in range(NPOOL)]
    hv = [rng.standard_normal((S, D)).astype(np.float16) for _ in range(NPOOL)]
    n_e2e = min(K, 16)
    barrier()
    t_e2e0 = time.perf_counter()
    for i in range(n_e2e):
        r = eng.decode_step(hq[i % NPOOL], hk[i % NPOOL], hv[i % NPOOL])
        if pg is not None:
            _ = pg.host()
        elif plan.needs_gather:
            _ = gather_outputs(torch.from_numpy(r.output).to(dev), plan).cpu()
    barrier()
    e2e_ms = (time.perf_counter() - t_e2e0) * 1000.0 / n_e2e
    vals = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
    if world > 1:
        vals = allreduce_max(vals)
    e2e_ms = float(vals[0])
    # e2e at the 256K point vs the device-timed last point: scale the growth
    # rate by the same host-path overhead
    e2e_value = value * curve[-1]["ms_per_step"] / e2e_ms

    st = eng.state()
    rec, payload = st["record_bytes"], st["payload_bytes"]
    slow_ms = curve[-1]["slow_kernel_ms"]
    achieved = union_last * payload / (slow_ms * 1e-3) / 1e9 if slow_ms > 0 else 0.0
    evict_bytes = S * rec  # one record per stream per eviction step
    ek = [c["evict_kernel_ms"] for c in curve if c["eviction_steps"]]
    evict_kernel_ms = statistics.mean(ek) if ek else None
    line = {
        "metric": metric_for(args.workload), "value": value, "unit": UNIT, "n_gpus": world,
        "steps": K * len(points), "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (device N(0,1) KV rounded to fp16, random queries)",
        "config": {
            "workload": w["desc"] + (f", head-sharded over {world} GPUs" if plan.needs_gather
                                     else ""),
            "output_gather": gather_kind,
            "growth_points": list(points), "steps_per_point": K,
            "timing": ("per point: one eviction period (B consecutive steps) timed with CUDA "
                       "events; value = 131072 tokens / trapezoid integral of ms/step over "
                       "the sampled 128K->256K curve"),
            "streams_per_gpu": S, "heads_per_stream": G, "batch": 1, "d": D, "block": B,
            "l_fast": L_FAST, "bits": "K8/V4", "fetch_fraction": FRAC,
            "selection": "group-shared" if args.group_select else "per-query-head (reference)",
            "slow_tier": "pinned host DRAM, zero-copy PCIe" if args.slow_tier == "host" else "HBM",
            "parallelism": f"heads-shard{world}" if world > 1 else "single",
            "l2": "inputs larger than L2 (slow tier 6.8-13.7 GB)",
        },
        "growth_curve": curve,
        "eviction": {"steps": len(evict_ms),
                     "step_ms_mean": statistics.mean(evict_ms) if evict_ms else None,
                     "non_eviction_step_ms_mean": statistics.mean(non_ev) if non_ev else None,
                     "evict_kernel_ms": evict_kernel_ms,
                     "d2h_bytes_per_eviction_step": evict_bytes,
                     "d2h_gbs": (evict_bytes / (evict_kernel_ms * 1e-3) / 1e9
                                 if evict_kernel_ms else None)},
        "roofline": {
            "bound": "pcie_h2d", "kernel": "slow_stream_attn", "at_ctx": curve[-1]["ctx_start"],
            "achieved": achieved, "peak": h2d_peak, "unit": "GB/s", "frac": achieved / h2d_peak,
            "peak_source": "pinned cudaMemcpy H2D 256 MiB best of 10, measured in this run" +
                           (", all ranks concurrently" if world > 1 else ""),
            "traffic": None, "algorithmic_bytes_per_launch": union_last * payload,
            "launch_ms": slow_ms},
        "kernel_ms_per_step": {k[3:]: v / (K * len(points)) for k, v in kt_tot.items()
                               if k.startswith("ms_")},
        "gpu_launches": launches,
        "e2e": {"value": e2e_value, "unit": UNIT,
                "h2d_bytes_per_step": hq[0].nbytes + hk[0].nbytes + hv[0].nbytes,
                "d2h_bytes_per_step": S * G * D * 8 * (world if plan.needs_gather else 1),
                "ms_per_step_at_last_point": e2e_ms,
                "note": "host-buffer C-ABI steps at the last point; value scaled by the "
                        "device/host step-time ratio there"},
        "prefill_s": round(prefill_s, 2),
    }
    if rank == 0:
        line["clocks"] = clk.summary()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            ctx = points[-1]
            total = S * G
            ms, _, engines, threads = ref_sample(ctx, 2, G,
                                                 engines=total if total <= 64 else None)
            line["cpu_baseline"] = {
                "value": cpu_throughput(float(ms[-1]), engines, total, 1), "unit": UNIT,
                "cores": threads, "kind": "reference",
                "sample": (f"{engines} unmodified reference Engines at {ctx} ctx (the end of the "
                           f"growth; upper bound on its sustained rate), 2 decode steps on "
                           f"{threads} threads (last timed: {ms[-1]:.0f} ms), "
                           f"{scale_note(engines, total)}")}
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": host_cores(),
                                    "kind": "reference", "sample": f"unavailable: {e}"}
    eng.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_layer_sequential(args):
    """Layer-sequential decode (--layer-sequential): a model's layers attend one
    after another (layer l+1's query depends on layer l's output), so one
    token is `layers` dependent decode calls, each over that layer's
    kv_heads x batch streams, on one CUDA stream.  One handle per layer; same
    data, metric and roofline as the batched step.  N = 1 only."""
    import numpy as np
    import torch
    import paper_2604_19769_b200 as T

    w = args.w
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    Lyr, G, ctx = w["layers"], w["G"], w["ctx"]
    S = w["kv_heads"] * w["batch"]
    cfg = T.TierConfig(hbm_budget_bytes=L_FAST * 2 * D * 2, d_k=D, d_v=D, bytes_full_precision=2,
                       block_size=B, key_bits=8, value_bits=4, fetch_fraction=FRAC)
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)
    engs = []
    for layer in range(Lyr):
        e = T.MultiStreamEngine(cfg, T.SelectionPolicy(None, FRAC), n_streams=S,
                                heads_per_stream=G, device=0,
                                reserve_tokens=ctx + args.warmup + args.steps + 2 * B,
                                slow_tier=0 if args.slow_tier == "host" else 1)
        e.set_stream(stream.cuda_stream)
        e.prefill_synthetic(ctx, seed=7000 + layer)
        engs.append(e)
    h2d_peak = measure_h2d_peak(torch, dev)
    gen = torch.Generator(device=dev).manual_seed(0)
    qs = [torch.randn(S, G, D, device=dev, generator=gen) for _ in range(Lyr)]
    ks = [torch.randn(S, D, device=dev, generator=gen).half() for _ in range(Lyr)]
    vs = [torch.randn(S, D, device=dev, generator=gen).half() for _ in range(Lyr)]
    outs = [torch.empty(S, G, D, device=dev, dtype=torch.float64) for _ in range(Lyr)]

    def token():
        for layer, e in enumerate(engs):
            e.decode_step_device(qs[layer].data_ptr(), ks[layer].data_ptr(), vs[layer].data_ptr(),
                                 outs[layer].data_ptr(), dtype=1)

    for _ in range(args.warmup):
        token()
    torch.cuda.synchronize()
    launches0 = sum(e.state()["launches"] for e in engs)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(0) as clk:
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(args.steps):
            token()
        ev1.record()
        torch.cuda.synchronize()
    ms_step = ev0.elapsed_time(ev1) / args.steps
    launches = sum(e.state()["launches"] for e in engs) - launches0
    union = sum(e.step_counters()[0] for e in engs)
    st = engs[0].state()
    pcie = union * st["payload_bytes"]
    host_tier = args.slow_tier == "host"
    hbm = sum(S * st["fast_tokens"] * 2 * D * 2 + S * st["slow_blocks"] * D * 4 for _ in engs) + \
        union * (st["record_bytes"] - st["payload_bytes"]) + (0 if host_tier else pcie)
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:  # noqa: BLE001
        pass
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    t_roof = max(hbm / (hbm_peak * 1e9), (pcie / (h2d_peak * 1e9)) if host_tier else 0.0) * 1e3
    line = {
        "metric": metric_for(args.workload) + ", layer-sequential", "value": w["batch"] * 1e3 / ms_step,
        "unit": UNIT, "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f32", "data": "synthetic (device N(0,1) KV rounded to fp16, random queries)",
        "config": {"workload": w["desc"] + f", layer-sequential: {Lyr} dependent calls per token",
                   "ctx": ctx, "streams_per_layer": S, "heads_per_stream": G,
                   "slow_tier": "pinned host DRAM, zero-copy PCIe" if host_tier else "HBM"},
        "ms_per_layer": ms_step / Lyr,
        "roofline": {"tier_roofline_ms": t_roof, "tier_frac": t_roof / ms_step,
                     "pcie_gbs": pcie / (ms_step * 1e-3) / 1e9 if host_tier else None,
                     "pcie_peak": h2d_peak},
        "clocks": clk.summary(),
        "gpu_launches": launches,
    }
    for e in engs:
        e.close()
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.layer_sequential:
        run_layer_sequential(args)
    elif args.workload == "cfg5":
        run_growth(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()
