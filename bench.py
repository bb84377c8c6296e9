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


def ctx_label(ctx):
    return f"{ctx // 1024}K" if ctx % 1024 == 0 else str(ctx)


def desc_for(name, ctx):
    """The workload description at the effective context (--ctx overrides)."""
    d = WORKLOADS[name]["desc"]
    base = ctx_label(WORKLOADS[name]["ctx"])
    return d if ctx == WORKLOADS[name]["ctx"] else d.replace(f"{base} ctx", f"{ctx_label(ctx)} ctx")


def metric_for(name, ctx):
    if name == "cfg2":
        return (f"decode tokens/s at {ctx_label(ctx)} ctx "
                "(LLaMA-3-8B GQA, all layers, batch 1)")
    return f"decode tokens/s ({desc_for(name, ctx)})"


def make_config(args, world, S):
    """The `config` object, identical in both arms for the same command line."""
    w = args.w
    mode = "heads" if w["batch"] == 1 else "requests"
    return {
        "workload": desc_for(args.workload, w["ctx"]) + (
            f", {mode}-sharded over {world} GPUs" if world > 1 else ""),
        "ctx": w["ctx"], "streams": w["layers"] * w["kv_heads"] * w["batch"],
        "streams_per_gpu": S, "heads_per_stream": w["G"], "batch": w["batch"], "d": D,
        "block": B, "l_fast": L_FAST, "bits": "K8/V4", "fetch_fraction": FRAC,
        "selection": "group-shared" if args.group_select else "per-query-head (reference)",
        "slow_tier": "pinned host DRAM, zero-copy PCIe" if args.slow_tier == "host" else "HBM",
        "parallelism": f"{mode}-shard{world}" if world > 1 else "single",
        "l2": "inputs larger than L2 (fp16 ring + slow tier far above 126 MB)",
    }


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
    if a.gpus < 1:
        p.error("--gpus must be >= 1")
    return a


def free_port():
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def self_launch(args):
    """`bench.py --gpus N` outside torchrun: launch N ranks (one process per
    GPU) under torch.distributed.run and exit with its status.  Fails loudly
    when fewer than N devices are visible (TTKV_SHARE_DEVICE=1 runs every rank
    on cuda:0 -- the test mode of the N>1 path on a one-GPU box)."""
    if args.impl == "ours" and os.environ.get("TTKV_SHARE_DEVICE") != "1":
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus:
            print(f"bench.py --gpus {args.gpus}: only {have} CUDA device(s) visible",
                  file=sys.stderr, flush=True)
            sys.exit(2)
    env = dict(os.environ)
    if os.environ.get("TTKV_DIST_BACKEND", "nccl") == "nccl":
        # communicator init on every rank stays visible in the log
        env.setdefault("NCCL_DEBUG", "INFO")
        env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    print("self-launch: " + " ".join(cmd), file=sys.stderr, flush=True)
    sys.exit(subprocess.call(cmd, env=env))


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
    """The reference arm: the unmodified reference engine (oracle/_ref) on the
    host cores.  Each step is a bounded sample -- `engines` of the workload's
    S x G reference Engines (one per (stream, query head)) decoding once on
    all host threads; the full step is that sample time x `factor`
    (total / sampled Engines, the Engines are independent).  `ms_per_step` and
    `steps` are what actually ran; `value` is the extrapolated throughput."""
    rank, _, world = dist_env()
    if rank != 0:
        return
    world = max(world, args.gpus)
    w = args.w
    S = w["layers"] * w["kv_heads"] * w["batch"]
    total_engines = S * w["G"]  # one reference Engine per (stream, q-head)
    n = args.warmup + args.steps
    # small workloads (cfg1: 32 Engines) run in full; larger ones are sampled
    ms, pre_s, engines, threads = ref_sample(w["ctx"], n, w["G"],
                                             engines=total_engines if total_engines <= 64 else None)
    timed = ms[args.warmup:]
    factor = total_engines / engines
    sample_ms = float(statistics.mean(timed))
    value = cpu_throughput(sample_ms, engines, total_engines, w["batch"])
    sample = (f"{engines} reference Engines (1 per stream x q-head) at {w['ctx']} ctx on "
              f"{threads} threads, {args.steps} timed decode steps after {args.warmup} warm-up; "
              f"{scale_note(engines, total_engines)}")
    line = {
        "impl": "reference", "metric": metric_for(args.workload, w["ctx"]), "value": value,
        "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": sample_ms, "higher_is_better": True,
        "scaling": "strong" if world > 1 and w["batch"] == 1 else "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (reference GaussianSource)",
        "config": make_config(args, world, S // world),
        "extrapolation": {
            "engines_sampled": engines, "engines_total": total_engines, "factor": factor,
            "sample_ms_per_step": sample_ms, "full_step_ms": sample_ms * factor,
            "note": "ms_per_step is the sample's wall time per step; value = tokens per full "
                    "step / (sample ms x factor)"},
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
    """SM clocks and throttle reasons sampled DURING the timed region: an NVML
    read when the region opens and closes plus a 10 ms sampler thread in
    between (nvidia-smi -lms 100 when NVML is unavailable).  A region shorter
    than ~50 ms cannot give 5 samples; `admissible` says whether it did."""
    REASONS = (("hw_slowdown", 0x8), ("sw_thermal_slowdown", 0x20),
               ("hw_thermal_slowdown", 0x40), ("sw_power_cap", 0x4))
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device):
        self.device = device
        self.samples = []  # (sm_mhz, max_mhz, reason bits)
        self.proc = None
        self.nvml = None
        self.source = None

    def _read(self):
        n = self.nvml
        sm = n.nvmlDeviceGetClockInfo(self.h, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(self.h, n.NVML_CLOCK_SM)
        try:
            rs = n.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        except Exception:  # noqa: BLE001 -- older bindings
            rs = n.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
        self.samples.append((float(sm), float(mx), int(rs)))

    def _loop(self):
        while not self._stop.wait(0.01):
            try:
                self._read()
            except Exception:  # noqa: BLE001
                return

    def __enter__(self):
        import threading
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nvml = pynvml
            try:
                self.h = pynvml.nvmlDeviceGetHandleByPciBusId(_bus_id(self.device).encode())
            except Exception:  # noqa: BLE001
                self.h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self._read()
            self._stop = threading.Event()
            self.th = threading.Thread(target=self._loop, daemon=True)
            self.th.start()
            self.source = "nvml 10 ms + region open/close"
        except Exception:  # noqa: BLE001
            self.nvml = None
            try:
                self.proc = subprocess.Popen(
                    ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                     "--format=csv,noheader,nounits", "-lms", "100"],
                    stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
                self.source = "nvidia-smi -lms 100"
            except Exception:  # noqa: BLE001
                self.proc = None
        return self

    def __exit__(self, *a):
        if self.nvml is not None:
            self._stop.set()
            self.th.join(timeout=1)
            try:
                self._read()
            except Exception:  # noqa: BLE001
                pass
        if self.proc:
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()
                out = ""
            names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
            bits = dict(self.REASONS)
            for l in out.splitlines():
                f = [x.strip() for x in l.split(",")]
                try:
                    sm, mx = float(f[1]), float(f[2])
                except (ValueError, IndexError):
                    continue
                rs = sum(bits[n] for n, v in zip(names, f[5:9]) if v.lower().startswith("active"))
                self.samples.append((sm, mx, rs))

    def summary(self):
        sm = [x[0] for x in self.samples]
        mx = max((x[1] for x in self.samples), default=None)
        reasons = sorted({n for _, _, r in self.samples for n, b in self.REASONS if r & b})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "sm_mhz_min": min(sm) if sm else None, "reasons": reasons,
                "samples": len(sm), "admissible": len(sm) >= 5, "source": self.source}


def _bus_id(device):
    """PCI bus id of a CUDA ordinal (the NVML handle of the same GPU)."""
    import ctypes as C_
    from paper_2604_19769_b200 import _lib as L
    buf = C_.create_string_buffer(32)
    if L.lib().ttkv_pci_bus_id(device, buf, 32) != 0:
        raise RuntimeError("pci bus id unavailable")
    return buf.value.decode()


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


def numa_nodes():
    try:
        return sorted(int(d[4:]) for d in os.listdir("/sys/devices/system/node")
                      if d.startswith("node") and d[4:].isdigit())
    except OSError:
        return [0]


def bind_numa(device):
    """Pin this rank to the CPUs of its GPU's NUMA node before the pinned
    slow-tier arena is allocated, so cudaHostAlloc's pages land on the node
    whose memory controller sits next to that GPU's PCIe root port (8-GPU
    boxes have two sockets; each rank streams ~51 GB/s from host DRAM).
    Returns what happened; on a multi-node host a failed binding is an error
    (the per-GPU PCIe numbers would mix remote-socket traffic)."""
    info = {"numa_nodes": len(numa_nodes()), "bound": False}
    try:
        bus = _bus_id(device).lower()
        info["bus_id"] = bus
        try:
            with open(f"/sys/bus/pci/devices/{bus}/numa_node") as f:
                info["gpu_numa_node"] = int(f.read().strip())
        except (OSError, ValueError):
            info["gpu_numa_node"] = None
        import pynvml
        pynvml.nvmlInit()
        try:
            h = pynvml.nvmlDeviceGetHandleByPciBusId(bus.encode())
        except Exception:  # noqa: BLE001
            h = pynvml.nvmlDeviceGetHandleByIndex(device)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, 16)
        cpus = {64 * i + b for i, w in enumerate(words) for b in range(64) if (w >> b) & 1}
        cpus &= os.sched_getaffinity(0)
        if cpus:
            os.sched_setaffinity(0, cpus)
            info["bound"] = True
            info["cpus"] = len(cpus)
    except Exception as e:  # noqa: BLE001
        info["error"] = repr(e)
        if info["numa_nodes"] > 1:
            raise RuntimeError(f"bind_numa: multi-socket host and the binding failed: {e!r}")
    return info


def init_dist(torch, dist, local, world):
    """One process per GPU: NCCL over NVLink.  TTKV_DIST_BACKEND=gloo with
    TTKV_SHARE_DEVICE=1 runs every rank on cuda:0 (exercises the N>1 path on a
    1-GPU box; the NVLink numbers need NCCL and one GPU per rank)."""
    share = os.environ.get("TTKV_SHARE_DEVICE") == "1"
    if world > 1 and not share and torch.cuda.device_count() < world:
        raise RuntimeError(f"{world} ranks but only {torch.cuda.device_count()} CUDA devices")
    dev = torch.device("cuda", 0 if share else local)
    numa = bind_numa(dev.index)
    torch.cuda.set_device(dev)
    if world > 1:
        backend = os.environ.get("TTKV_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)
    return dev, numa


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
            pg = PeerGather(eng, plan)
            return pg, ("combine fused with the all-gather over peer memory "
                        f"(P2P probe OK for all {plan.world} ranks)")
        except Exception as e:  # noqa: BLE001
            print(f"peer gather unavailable ({e}); using NCCL all_gather", file=sys.stderr,
                  flush=True)
            return None, f"NCCL all_gather (peer gather unavailable: {e})"
    return None, "NCCL all_gather (TTKV_GATHER=nccl)"


def traffic_for(kernel, workload):
    """DRAM (and PCIe sysmem) traffic per launch of the dominant kernel from
    its committed `ncu --set full` capture (profiles/traffic.json, written by
    tools/stamp_traffic.py), reported only while the loaded kernel's SASS
    signature equals the measured one; otherwise null with fresh=false."""
    t = (load_traffic() or {}).get(f"{kernel}@{workload}")
    try:
        sys.path.insert(0, os.path.join(ROOT, "tools"))
        import kernel_sig
        cur = kernel_sig.kernel_sig(kernel)
    except Exception as e:  # noqa: BLE001 -- cuobjdump missing: cannot prove freshness
        cur = f"unavailable: {e}"
    if not t:
        return None, None, {"source": None, "fresh": False, "loaded_sig": cur}
    fresh = t.get("sig") is not None and t.get("sig") == cur
    meta = {"source": t.get("source"), "git": t.get("git"), "sig": t.get("sig"),
            "loaded_sig": cur, "fresh": fresh}
    if not fresh:
        return None, None, meta
    return t.get("dram_bytes_per_launch"), t.get("sysmem_read_bytes_per_launch"), meta


def read_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:  # noqa: BLE001
        return {}


def fast_tier_solo(T, cfg, S, G, dev, stream, args, torch):
    """The fast-tier kernel timed alone (no slow work on the GPU beside it): a
    second handle with the same S x L_FAST fp16 ring and no slow tier yet."""
    n_kt = 5
    e = T.MultiStreamEngine(cfg, T.SelectionPolicy(None, FRAC), n_streams=S, heads_per_stream=G,
                            device=dev.index, reserve_tokens=L_FAST + 2 * B)
    e.set_stream(stream.cuda_stream)
    e.prefill_synthetic(L_FAST - 3 - n_kt, seed=99)
    gen = torch.Generator(device=dev).manual_seed(123)
    q = torch.randn(S, G, D, device=dev, generator=gen)
    k = torch.randn(S, D, device=dev, generator=gen).half()
    v = torch.randn(S, D, device=dev, generator=gen).half()
    o = torch.empty(S, G, D, device=dev, dtype=torch.float64)
    for _ in range(2):
        e.decode_step_device(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), dtype=1)
    torch.cuda.synchronize()
    f0 = e.state()["fast_tokens"]
    e.kernel_times(reset=True)
    e.set_timing(True)
    for _ in range(n_kt):
        e.decode_step_device(q.data_ptr(), k.data_ptr(), v.data_ptr(), o.data_ptr(), dtype=1)
    torch.cuda.synchronize()
    e.set_timing(False)
    kt = e.kernel_times(reset=True)
    assert e.state()["slow_blocks"] == 0
    e.close()
    ms = kt["ms_fast"] / max(1, kt["n_fast"])
    F = f0 + (n_kt + 1) / 2.0  # mean fast-tier length over the timed steps
    byts = S * F * 2 * D * 2
    return {"ms": ms, "tokens": F, "bytes": byts, "hbm_gbs": byts / (ms * 1e-3) / 1e9,
            "note": "fast_attn timed alone: a handle with the same S x L_FAST ring, no slow tier"}


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist
    import paper_2604_19769_b200 as T
    from paper_2604_19769_b200.sharding import ShardPlan, gather_outputs

    rank, local, world = dist_env()
    dev, numa = init_dist(torch, dist, local, world)
    w = args.w
    G, ctx, batch = w["G"], w["ctx"], w["batch"]
    mode = "heads" if batch == 1 else "requests"
    plan = ShardPlan(rank, world, w["layers"], w["kv_heads"], batch, mode)
    S = plan.n_local  # streams on this rank
    host_tier = args.slow_tier == "host"

    cfg = T.TierConfig(hbm_budget_bytes=L_FAST * 2 * D * 2, d_k=D, d_v=D, bytes_full_precision=2,
                       block_size=B, key_bits=8, value_bits=4, fetch_fraction=FRAC)
    max_steps = args.steps if args.steps_given else 2000
    n_steps_total = args.warmup + 2 * max_steps + 16  # timed + kernel-breakdown + e2e steps
    eng = T.MultiStreamEngine(cfg, T.SelectionPolicy(None, FRAC), n_streams=S,
                              heads_per_stream=G, group_select=args.group_select, device=dev.index,
                              reserve_tokens=ctx + n_steps_total + B,
                              slow_tier=0 if host_tier else 1)
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
        if i == 0 and pg is not None:
            # the fused peer-memory gather must reproduce the collective before
            # it is timed; otherwise every rank falls back to NCCL together
            ok, why = pg.verify(out)
            if ok:
                gather_kind += "; first step bit-identical to the collective's all-gather"
            else:
                pg.close()
                pg = None
                gather_kind = f"NCCL all_gather (peer gather self-check failed: {why})"
                print(gather_kind, file=sys.stderr, flush=True)
    barrier()
    if not args.steps_given:
        # default K: at least 10 steps and >= ~1 s of timed region (clock samples)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step(args.warmup)
        e1.record()
        barrier()
        one = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
        one = float(allreduce_max(one)[0]) if world > 1 else float(one[0])
        args.steps = int(min(max_steps, max(10, -(-1000.0 // max(one, 1e-3)))))
    base = args.warmup + 1
    st0 = eng.state()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev.index) as clk:
        barrier()
        ev0.record()
        for i in range(args.steps):
            step(base + i)
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
        step(base + args.steps + i)
    barrier()
    eng.set_timing(False)
    kt = eng.kernel_times(reset=True)

    # --- e2e through the public C ABI with host buffers -----------------------
    pins, hq, hk, hv, hout = pinned_step_buffers(np.random.default_rng(rank), S, G, NPOOL)
    h2d = hq[0].nbytes + hk[0].nbytes + hv[0].nbytes
    d2h = S * G * D * 8 * (world if plan.needs_gather else 1)
    barrier()
    t_e2e0 = time.perf_counter()
    for i in range(args.steps):
        r = eng.decode_step(hq[i % NPOOL], hk[i % NPOOL], hv[i % NPOOL], out=hout)
        if pg is not None:
            _ = pg.host()
        elif plan.needs_gather:
            _ = gather_outputs(torch.from_numpy(r.output).to(dev), plan).cpu()
    barrier()
    e2e_ms = (time.perf_counter() - t_e2e0) * 1000.0 / args.steps

    # --- roofline of the dominant kernel ----------------------------------------
    rec = st1["record_bytes"]
    payload = st1["payload_bytes"]  # params are staged from the HBM mirror
    slow_ms = kt["ms_slow"] / max(1, kt["n_slow"])
    pcie_bytes_launch = union_last * payload
    achieved = pcie_bytes_launch / (slow_ms * 1e-3) / 1e9 if slow_ms > 0 else 0.0
    F = st1["fast_tokens"]
    fast_bytes = S * F * 2 * D * 2
    fast_conc_ms = kt["ms_fast"] / max(1, kt["n_fast"])
    hbm_peak = read_peaks().get("hbm_gbs", 6650.0)
    hbm_bytes_step = fast_bytes + S * st1["slow_blocks"] * D * 4 + union_last * (rec - payload)
    fast_solo = fast_tier_solo(T, cfg, S, G, dev, stream, args, torch)
    fast_solo.update({"hbm_peak": hbm_peak, "frac": fast_solo["hbm_gbs"] / hbm_peak,
                      "peak_source": "MEASURED_PEAKS.json hbm_gbs",
                      "concurrent_ms": fast_conc_ms,
                      "concurrent_note": "wall time on the low-priority stream beside the slow "
                                         "kernel (hidden under it), not an HBM rate"})

    # --- per-rank facts and the max over ranks ----------------------------------
    me = {"rank": rank, "device": dev.index, "numa": numa, "h2d_peak_gbs": h2d_peak,
          "union_blocks": union_last, "pcie_bytes": pcie_bytes_launch if host_tier else 0,
          "slow_kernel_ms": slow_ms, "pcie_gbs": achieved if host_tier else None,
          "ms_timed": ms_total, "e2e_ms": e2e_ms}
    ranks = [me]
    if world > 1:
        ranks = [None] * world
        dist.all_gather_object(ranks, me)
    ms_total = max(r_["ms_timed"] for r_ in ranks)
    e2e_ms = max(r_["e2e_ms"] for r_ in ranks)
    ms_step = ms_total / args.steps
    tokens_per_step = batch  # one generated token per request per step
    value = tokens_per_step * 1000.0 / ms_step
    pcie_all = sum(r_["pcie_bytes"] for r_ in ranks)

    if host_tier:  # records cross PCIe (zero-copy); params + centroids + fast tier from HBM
        t_roof_ms = max(hbm_bytes_step / (hbm_peak * 1e9),
                        pcie_bytes_launch / (h2d_peak * 1e9)) * 1e3
        traffic, pcie_traffic, tmeta = traffic_for("slow_attn_kernel", args.workload)
        roof = {"bound": "pcie_h2d", "kernel": "slow_attn_kernel", "achieved": achieved,
                "peak": h2d_peak, "unit": "GB/s", "frac": achieved / h2d_peak,
                "peak_source": "pinned cudaMemcpy H2D 256 MiB best of 10, measured in this run" +
                               (", all ranks concurrently" if world > 1 else ""),
                "traffic": traffic, "pcie_traffic": pcie_traffic,
                "algorithmic_bytes_per_launch": pcie_bytes_launch}
    else:  # HBM-resident slow tier: every byte of the step is an HBM byte
        hbm_bytes_step += pcie_bytes_launch
        t_roof_ms = hbm_bytes_step / (hbm_peak * 1e9) * 1e3
        slow_bytes = union_last * rec  # payload from the arena + params from the mirror
        ach = slow_bytes / (slow_ms * 1e-3) / 1e9 if slow_ms > 0 else 0.0
        kname = ("slow_attn_tc5_kernel" if os.environ.get("TTKV_SLOW_TC5") == "1"
                 else "slow_attn_tc_kernel")  # the opt-in tcgen05 kernel has no stamped traffic
        traffic, _, tmeta = traffic_for(kname, args.workload)
        roof = {"bound": "hbm", "kernel": kname, "achieved": ach,
                "peak": hbm_peak, "unit": "GB/s", "frac": ach / hbm_peak,
                "peak_source": "MEASURED_PEAKS.json hbm_gbs (burst copy)", "traffic": traffic,
                "algorithmic_bytes_per_launch": slow_bytes}
        pcie_bytes_launch = 0

    line = {
        "metric": metric_for(args.workload, ctx), "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 and mode == "heads" else "weak", "vs_baseline": None,
        "dtype": "f32",
        "data": "synthetic (device N(0,1) KV rounded to fp16, random queries)",
        "config": make_config(args, world, S),
        "output_gather": gather_kind,
        "storage": "fp16 ring, u8 keys / u4 values, f32 params",
        "roofline": {
            **roof, "traffic_source": tmeta,
            "launch_ms": slow_ms,
            "tier_roofline_ms": t_roof_ms, "tier_frac": t_roof_ms / ms_step,
            "fast_attn": fast_solo,
        },
        "pcie_bytes_per_token": pcie_all / tokens_per_step,
        "union_blocks_per_step": sum(r_["union_blocks"] for r_ in ranks),
        "kernel_ms_per_step": {k[3:]: v / n_kt for k, v in kt.items() if k.startswith("ms_")},
        "gpu_launches": launches,
        "e2e": {"value": tokens_per_step * 1000.0 / e2e_ms, "unit": UNIT,
                "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms,
                "host_buffers": "page-locked caller buffers, read and written in place by the step's kernels (ttkv_gpu_decode_step)"},
        "prefill_s": round(prefill_s, 2),
    }
    if world > 1:
        line["ranks"] = ranks
    else:
        line["numa"] = numa
    if rank == 0:
        line["clocks"] = clk.summary()
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline_line(ctx, G, S * G, tokens_per_step)
    eng.close()
    if rank == 0:
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def pinned_step_buffers(rng, S, G, npool):
    """The e2e leg's host buffers: `npool` sets of random q [S, G, D] f32 and
    k, v [S, D] f16 plus one f64 output [S, G, D], all page-locked (numpy views
    of pinned torch tensors), so every step's H2D and D2H is a DMA from / to
    pinned host memory with no staging copy.  Returns (keep-alive, q, k, v, out)."""
    import numpy as np
    import torch

    def pinned(a):
        t = torch.empty(a.shape, dtype={np.float32: torch.float32, np.float16: torch.float16,
                                        np.float64: torch.float64}[a.dtype.type],
                        pin_memory=True)
        v = t.numpy()
        v[...] = a
        return t, v
    keep, qs, ks, vs = [], [], [], []
    for _ in range(npool):
        for dst, a in ((qs, rng.standard_normal((S, G, D)).astype(np.float32)),
                       (ks, rng.standard_normal((S, D)).astype(np.float16)),
                       (vs, rng.standard_normal((S, D)).astype(np.float16))):
            t, v = pinned(a)
            keep.append(t)
            dst.append(v)
    t, out = pinned(np.zeros((S, G, D), np.float64))
    keep.append(t)
    return keep, qs, ks, vs, out


def cpu_baseline_line(ctx, G, total, tokens_per_step, warm=2, timed=5, note=""):
    """The unmodified reference engine on this box's host cores: `timed`
    decode steps after `warm` of a bounded sample of Engines, extrapolated."""
    try:
        ms, _, engines, threads = ref_sample(ctx, warm + timed, G,
                                             engines=total if total <= 64 else None)
        m = float(statistics.mean(ms[warm:]))
        return {
            "value": cpu_throughput(m, engines, total, tokens_per_step), "unit": UNIT,
            "cores": threads, "kind": "reference",
            "sample": (f"{engines} unmodified reference Engines at {ctx} ctx{note}, {timed} "
                       f"decode steps timed after {warm} on {threads} threads (mean {m:.0f} ms), "
                       f"{scale_note(engines, total)}"),
            "sample_ms_per_step": [round(float(x), 1) for x in ms[warm:]]}
    except Exception as e:  # noqa: BLE001
        return {"value": None, "unit": UNIT, "cores": host_cores(), "kind": "reference",
                "sample": f"unavailable: {e}"}


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
    dev, numa = init_dist(torch, dist, local, world)
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
    pins, hq, hk, hv, hout = pinned_step_buffers(np.random.default_rng(rank), S, G, NPOOL)
    n_e2e = min(K, 16)
    barrier()
    t_e2e0 = time.perf_counter()
    for i in range(n_e2e):
        r = eng.decode_step(hq[i % NPOOL], hk[i % NPOOL], hv[i % NPOOL], out=hout)
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
    growth_traffic = traffic_for("slow_attn_kernel", "cfg5")
    ek = [c["evict_kernel_ms"] for c in curve if c["eviction_steps"]]
    evict_kernel_ms = statistics.mean(ek) if ek else None
    line = {
        "metric": metric_for(args.workload, points[-1]), "value": value, "unit": UNIT,
        "n_gpus": world, "steps": K * len(points), "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True,
        "scaling": "strong" if world > 1 else "weak", "vs_baseline": None, "dtype": "f32",
        "data": "synthetic (device N(0,1) KV rounded to fp16, random queries)",
        "output_gather": gather_kind,
        "config": {
            **make_config(args, world, S),
            "growth_points": list(points), "steps_per_point": K,
            "timing": ("per point: one eviction period (B consecutive steps) timed with CUDA "
                       "events; value = 131072 tokens / trapezoid integral of ms/step over "
                       "the sampled 128K->256K curve"),
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
            "traffic": growth_traffic[0], "pcie_traffic": growth_traffic[1],
            "traffic_source": growth_traffic[2],
            "algorithmic_bytes_per_launch": union_last * payload,
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
        line["cpu_baseline"] = cpu_baseline_line(
            points[-1], G, S * G, 1,
            note=" (the end of the growth; upper bound on its sustained rate)")
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
    args.max_auto = args.steps if args.steps_given else 2000
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
                                reserve_tokens=ctx + args.warmup + args.max_auto + 2 * B,
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
    if not args.steps_given:  # >= 10 tokens and >= ~1 s of timed region
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        token()
        e1.record()
        torch.cuda.synchronize()
        args.steps = int(min(args.max_auto, max(10, -(-1000.0 // max(e0.elapsed_time(e1), 1e-3)))))
    launches0 = sum(e.state()["launches"] for e in engs)
    spec0 = sum(e.state()["spec_steps"] for e in engs)
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
    spec_calls = sum(e.state()["spec_steps"] for e in engs) - spec0
    union = sum(e.step_counters()[0] for e in engs)
    st = engs[0].state()
    # speculative record stream (HBM tier): every record of the layer streamed
    # beside the selection; the roofline keeps the union's (algorithmic) bytes
    streamed = sum(S * e.state()["slow_blocks"] for e in engs) if spec_calls else union
    pcie = union * st["payload_bytes"]
    host_tier = args.slow_tier == "host"
    hbm = sum(S * st["fast_tokens"] * 2 * D * 2 + S * st["slow_blocks"] * D * 4 for _ in engs) + \
        union * (st["record_bytes"] - st["payload_bytes"]) + (0 if host_tier else pcie)
    hbm_peak = read_peaks().get("hbm_gbs", 6650.0)
    t_roof = max(hbm / (hbm_peak * 1e9), (pcie / (h2d_peak * 1e9)) if host_tier else 0.0) * 1e3
    line = {
        "metric": metric_for(args.workload, ctx) + ", layer-sequential",
        "value": w["batch"] * 1e3 / ms_step,
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
        "record_stream": ("speculative: every record, beside the selection "
                          "(slow_attn_tc_spec_kernel)") if spec_calls else "union after the selection",
        "spec_calls_frac": spec_calls / float(args.steps * Lyr),
        "records_per_token": {"union": union, "streamed": streamed},
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
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ and args.impl == "ours":
        if args.layer_sequential:
            sys.exit("--layer-sequential runs on one GPU")
        self_launch(args)
    if "WORLD_SIZE" in os.environ and int(os.environ["WORLD_SIZE"]) != args.gpus:
        sys.exit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ['WORLD_SIZE']}")
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
