"""The reference harness on the B200 engine, with measured timelines.

Mirrors /root/reference/proj/core/src/harness.cpp (run_benchmark 88-171,
run_sweep 173-208, run_ablation 210-221, report writers 225-322) with one
change of meaning: the latency columns are measured B200 device time of
each decode step (CUDA events on the engine's critical-path stream) instead
of the analytic two-lane simulator (sim.cpp).  Baseline emulation follows
effective_tier_config / effective_policy / serial_schedule (harness.cpp:22-24,
56-86); the serial baselines run the engine's bulk schedule (all selected
records cross PCIe into HBM before any attention).  H->G bytes use the
reference's modeled accounting, so traffic columns are comparable with the
reference byte for byte; the actual PCIe bytes are reported beside them.
"""
from __future__ import annotations

import ctypes as C
import json
import math
import os
import re
from dataclasses import dataclass, field, replace
from typing import List, Optional

import numpy as np

from . import _lib as L
from .engine import (ConfigError, IoError, MultiStreamEngine, SelectionPolicy, TierConfig,
                     fast_capacity)

BASELINES = ("ttkv", "fp16_full_fetch", "uniform_quant_8_8", "no_pipeline", "single_tier")
ABLATION_ORDER = ("fp16_full_fetch", "single_tier", "uniform_quant_8_8", "no_pipeline", "ttkv")
KNEEDLE_SPAN = 128  # workload.hpp:10


@dataclass
class WorkloadSpec:
    """workload.hpp:15-35"""
    kind: str = "gaussian"  # or "needle"
    context_length: int = 4096
    decode_steps: int = 32
    d_k: int = 64
    d_v: int = 64
    seed: int = 0
    needle_block_position: int = 2
    needle_alignment_strength: float = 3.0


@dataclass
class RunRecord:
    method: str
    spec: WorkloadSpec
    tier: TierConfig
    policy: SelectionPolicy
    latency_ms: List[float] = field(default_factory=list)       # measured, per step
    step_bytes: List[float] = field(default_factory=list)       # modeled H->G
    baseline_bytes: List[float] = field(default_factory=list)   # fp16 full fetch
    pcie_bytes: List[int] = field(default_factory=list)         # measured record bytes
    blocks_scored: List[int] = field(default_factory=list)
    blocks_fetched: List[int] = field(default_factory=list)
    evictions: List[bool] = field(default_factory=list)
    oracle_errors: List[float] = field(default_factory=list)
    needle_hits: int = 0
    timelines: List[list] = field(default_factory=list)  # measured, per step
    summary: dict = field(default_factory=dict)


def _dropin_lib():
    path = os.path.join(os.path.dirname(L.LIB_PATH), "libttkv.so")
    lib = C.CDLL(path)
    f = lib.ttkv_generate_workload
    f.restype = C.c_int
    f.argtypes = [C.c_int, C.c_uint64, C.c_uint64, C.c_uint32, C.c_uint32, C.c_uint64,
                  C.c_uint64, C.c_double] + [C.c_void_p] * 5
    return lib


def generate_workload(spec: WorkloadSpec):
    """generate_workload (workload.cpp:42-95) through libttkv.so."""
    ctx, T, dk, dv = spec.context_length, spec.decode_steps, spec.d_k, spec.d_v
    arrs = [np.zeros((max(ctx, 1), dk), np.float32), np.zeros((max(ctx, 1), dv), np.float32),
            np.zeros((max(T, 1), dk), np.float32), np.zeros((max(T, 1), dv), np.float32),
            np.zeros((max(T, 1), dk), np.float32)]
    rc = _dropin_lib().ttkv_generate_workload(
        int(spec.kind == "needle"), ctx, T, dk, dv, spec.seed, spec.needle_block_position,
        spec.needle_alignment_strength, *[a.ctypes.data_as(C.c_void_p) for a in arrs])
    if rc != 0:
        raise ValueError("invalid workload spec")
    pk, pv, dk_, dv_, dq = arrs
    return pk[:ctx], pv[:ctx], dk_[:T], dv_[:T], dq[:T]


def effective(tier: TierConfig, policy: SelectionPolicy, baseline: str):
    """effective_tier_config / effective_policy / serial_schedule
    (harness.cpp:22-24, 56-86)."""
    if baseline not in BASELINES:
        raise ValueError(f"unknown baseline {baseline}")
    t = replace(tier)
    if t.hbm_budget_bytes == 0:
        t.hbm_budget_bytes = 1024 * t.d_kv() * t.bytes_full_precision
    if baseline == "fp16_full_fetch":
        t.key_bits = t.value_bits = 16
    elif baseline == "uniform_quant_8_8":
        t.key_bits = t.value_bits = 8
    elif baseline == "single_tier":
        t.hbm_budget_bytes = t.block_bytes_full_precision()
    t.validate()
    p = SelectionPolicy(None, 1.0) if baseline in ("fp16_full_fetch", "single_tier") else policy
    serial = baseline in ("fp16_full_fetch", "no_pipeline")
    return t, p, serial


def _dense(q, keys, values):
    """reference::dense_attention (reference.cpp:12-41) in float64."""
    lg = keys.astype(np.float64) @ q.astype(np.float64) / math.sqrt(q.shape[0])
    w = np.exp(lg - lg.max())
    return (w[:, None] * values.astype(np.float64)).sum(0) / w.sum()


def _rel(a, b):
    den = float(np.sqrt((b * b).sum()))
    num = float(np.sqrt(((a - b) ** 2).sum()))
    return num / den if den > 0 else num


def aggregate(rec: RunRecord) -> dict:
    """aggregate_run (sim.cpp:152-184) over measured latencies."""
    lat = rec.latency_ms
    warm = 5 if len(lat) >= 25 else 0
    xs = sorted(lat[warm:])
    rank = math.ceil(0.95 * len(xs)) if xs else 0
    total = sum(lat[warm:])
    h2g = sum(rec.step_bytes)
    base = sum(rec.baseline_bytes)
    if h2g > 0:
        red = base / h2g
    else:
        red = math.inf if base > 0 else 1.0
    return dict(steps=len(lat), p95_latency_ms=xs[max(rank - 1, 0)] if xs else 0.0,
                mean_latency_ms=total / max(1, len(lat) - warm),
                tokens_per_second=(len(lat) - warm) / (total / 1e3) if total > 0 else 0.0,
                total_h2g_bytes=h2g, traffic_reduction=red,
                pcie_bytes_measured=int(sum(rec.pcie_bytes)))


def run_benchmark(tier: TierConfig, policy: SelectionPolicy, spec: WorkloadSpec,
                  baseline: str = "ttkv", oracle: bool = True, device: int = 0) -> RunRecord:
    """run_benchmark (harness.cpp:88-171) on the B200 engine."""
    t, p, serial = effective(tier, policy, baseline)
    l_fast = fast_capacity(t)
    pk, pv, dk, dv, dq = generate_workload(spec)
    if spec.kind == "needle":
        slow_after = 0 if spec.context_length <= l_fast else \
            ((spec.context_length - l_fast - 1) // t.block_size + 1) * t.block_size
        if (spec.needle_block_position + 1) * KNEEDLE_SPAN > slow_after:
            raise ValueError("needle span does not land in the slow tier for this config")
    # fp32 ring: the reference stores float32 tokens (kv_types.hpp:14-15)
    eng = MultiStreamEngine(t, p, n_streams=1, heads_per_stream=1, device=device,
                            reserve_tokens=spec.context_length + spec.decode_steps,
                            ring_bytes=4, serial_schedule=serial)
    rec = RunRecord(method=baseline, spec=spec, tier=t, policy=p)
    try:
        if spec.context_length:
            eng.prefill(pk[None], pv[None])
        hist_k, hist_v = list(pk), list(pv)
        eng.set_timing(True)
        eng.kernel_times(reset=True)
        needle_first = spec.needle_block_position * KNEEDLE_SPAN
        for s in range(spec.decode_steps):
            st = eng.state()
            rec.baseline_bytes.append(st["slow_blocks"] * t.block_size * t.d_kv() *
                                      t.bytes_full_precision)
            r = eng.decode_step(dq[s][None, None], dk[s][None], dv[s][None], fetched=True)
            kt = eng.kernel_times(reset=True)
            rec.latency_ms.append(kt["last_step_ms"])
            rec.timelines.append(eng.timeline())
            rec.step_bytes.append(r.bytes_transferred)
            rec.pcie_bytes.append(r.pcie_bytes)
            rec.blocks_scored.append(r.blocks_scored)
            rec.blocks_fetched.append(r.blocks_fetched)
            rec.evictions.append(r.eviction_occurred)
            hist_k.append(dk[s])
            hist_v.append(dv[s])
            if oracle:
                rec.oracle_errors.append(_rel(r.output[0, 0], _dense(dq[s], np.asarray(hist_k),
                                                                     np.asarray(hist_v))))
            if spec.kind == "needle" and st["slow_blocks"] * t.block_size > needle_first:
                if (needle_first // t.block_size) in set(int(x) for x in r.fetched_blocks[0][0]):
                    rec.needle_hits += 1
    finally:
        eng.close()
    rec.summary = aggregate(rec)
    return rec


# ---------------------------------------------------------------------------
# RunConfig files (harness.cpp:324-413): `key = value` lines, `#` comments.
# ---------------------------------------------------------------------------
@dataclass
class RunConfig:
    """harness.hpp:33-40"""
    tier: TierConfig = field(default_factory=TierConfig)
    policy: SelectionPolicy = field(default_factory=SelectionPolicy)
    baseline: str = "ttkv"
    format: str = "csv"
    out_dir: str = "."
    literal_merge: bool = False


_INT_RE = re.compile(r"\s*([+-]?)(\d+)")
_FLT_RE = re.compile(r"\s*([+-]?(?:(?:\d+\.?\d*|\.\d+)(?:[eE][+-]?\d+)?|inf(?:inity)?|nan))",
                     re.IGNORECASE)


def _stoull(v: str) -> int:
    """std::stoull: longest base-10 prefix after whitespace, a leading '-'
    negates modulo 2^64; no digits -> invalid_argument; > 2^64-1 -> out_of_range."""
    m = _INT_RE.match(v)
    if not m:
        raise ValueError("invalid")
    x = int(m.group(2))
    if x > 2 ** 64 - 1:
        raise OverflowError("range")
    return (2 ** 64 - x) % 2 ** 64 if m.group(1) == "-" else x


def _stod(v: str) -> float:
    """std::stod: longest decimal-float prefix; overflow -> out_of_range."""
    m = _FLT_RE.match(v)
    if not m:
        raise ValueError("invalid")
    x = float(m.group(1))
    if math.isinf(x) and "inf" not in m.group(1).lower():
        raise OverflowError("range")
    return x


def parse_config_file(path) -> dict:
    """parse_config_file (harness.cpp:324-346)."""
    try:
        with open(path, "r", newline="") as f:
            text = f.read()
    except OSError:
        raise IoError(f"cannot open config file {path}") from None
    values = {}
    lines = text.split("\n")
    if lines and lines[-1] == "":
        lines.pop()
    for lineno, line in enumerate(lines, 1):
        line = line.split("#", 1)[0].strip(" \t\r")
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"{path}:{lineno}: expected key = value")
        k, v = line.split("=", 1)
        values[k.strip(" \t\r")] = v.strip(" \t\r")
    return values


def apply_config_values(values: dict, config: RunConfig, spec: WorkloadSpec) -> None:
    """apply_config_values (harness.cpp:348-413); keys in std::map order."""
    u32 = lambda x: x % 2 ** 32  # static_cast<unsigned>(std::stoul(value))  # noqa: E731
    for key in sorted(values):
        value = values[key]
        try:
            if key == "seed": spec.seed = _stoull(value)  # noqa: E701
            elif key == "context_length": spec.context_length = _stoull(value)  # noqa: E701
            elif key == "decode_steps": spec.decode_steps = _stoull(value)  # noqa: E701
            elif key == "d_k": spec.d_k = _stoull(value)  # noqa: E701
            elif key == "d_v": spec.d_v = _stoull(value)  # noqa: E701
            elif key == "workload":
                if value == "gaussian":
                    spec.kind = "gaussian"
                elif value == "planted_needle":
                    spec.kind = "needle"
                else:
                    raise ConfigError("unknown workload kind: " + value)
            elif key == "needle_block_position": spec.needle_block_position = _stoull(value)  # noqa
            elif key == "needle_alignment_strength":
                spec.needle_alignment_strength = _stod(value)
            elif key == "hbm_budget_bytes": config.tier.hbm_budget_bytes = _stoull(value)  # noqa
            elif key == "block_size": config.tier.block_size = _stoull(value)  # noqa: E701
            elif key == "key_bits": config.tier.key_bits = u32(_stoull(value))  # noqa: E701
            elif key == "value_bits": config.tier.value_bits = u32(_stoull(value))  # noqa: E701
            elif key == "bytes_full_precision":
                config.tier.bytes_full_precision = _stoull(value)
            elif key == "fetch_fraction":
                config.tier.fetch_fraction = _stod(value)
                config.policy.fetch_fraction = _stod(value)
            elif key == "top_k_blocks":
                config.tier.top_k_blocks = _stoull(value)
                config.policy.top_k = _stoull(value)
            elif key == "hbm_bandwidth": config.tier.hbm_bandwidth = _stod(value)  # noqa: E701
            elif key == "pcie_bandwidth": config.tier.pcie_bandwidth = _stod(value)  # noqa: E701
            elif key == "transfer_latency": config.tier.transfer_latency = _stod(value)  # noqa
            elif key == "compute_rate": config.tier.compute_rate = _stod(value)  # noqa: E701
            elif key == "baseline":
                if value not in BASELINES:
                    raise ConfigError("unknown baseline: " + value)
                config.baseline = value
            elif key == "format":
                if value not in ("csv", "json"):
                    raise ConfigError("unknown format: " + value)
                config.format = value
            elif key == "out_dir": config.out_dir = value  # noqa: E701
            elif key == "literal_merge": config.literal_merge = value in ("1", "true")  # noqa
            else:
                raise ConfigError("unknown config key: " + key)
        except ValueError:
            raise ConfigError(f"bad value for {key}: {value}") from None
        except OverflowError:
            raise ConfigError(f"value out of range for {key}: {value}") from None


def load_run_config(path, config: Optional[RunConfig] = None,
                    spec: Optional[WorkloadSpec] = None):
    """Defaults < file (ttkv_bench.cpp:9): returns (RunConfig, WorkloadSpec)."""
    config = config or RunConfig()
    spec = spec or WorkloadSpec()
    apply_config_values(parse_config_file(path), config, spec)
    return config, spec


# ---------------------------------------------------------------------------
# The reference's two-lane timing model (sim.cpp:16-141), restated, and its
# calibration against measured B200 kernel times.
# ---------------------------------------------------------------------------
@dataclass
class LinkModel:
    """sim.hpp:12-15"""
    bandwidth: float = 3.2e10   # bytes/s
    fixed_latency: float = 0.0  # s per transfer


@dataclass
class Timeline:
    """PipelineTimeline (sim.hpp:35-46) without the per-event list."""
    total_latency: float = 0.0
    total_compute: float = 0.0
    total_transfer: float = 0.0
    idle_fraction: float = 0.0
    mean_transfer_stall: float = 0.0


def _sim(compute, transfers, link: LinkModel, rate: float, pipelined: bool) -> Timeline:
    """simulate_serial / simulate_pipelined (sim.cpp:90-141).  compute: list of
    amounts (elements) in schedule order; transfers: list of (compute index,
    bytes) in transfer order."""
    if link.bandwidth <= 0 or rate <= 0:
        raise ValueError("simulate: bandwidth and compute_rate must be positive")
    if link.fixed_latency < 0:
        raise ValueError("simulate: fixed_latency must be non-negative")
    tl = Timeline()
    finish = {}
    t = 0.0
    for ci, amount in transfers:  # transfer_finish_map (sim.cpp:32-45)
        t += link.fixed_latency + amount / link.bandwidth
        finish[ci] = t
    tl.total_transfer = t
    starts, lane = [], (tl.total_transfer if not pipelined else 0.0)
    for i, amount in enumerate(compute):
        start = max(lane, finish[i]) if (pipelined and i in finish) else lane
        dur = amount / rate
        starts.append(start)
        lane = start + dur
        tl.total_compute += dur
    tl.total_latency = max(lane, tl.total_transfer) if pipelined else lane
    ideal, t = [], 0.0  # ideal_starts (sim.cpp:49-57)
    for amount in compute:
        ideal.append(t)
        t += amount / rate
    stalls = [starts[i] - ideal[i] for i in range(len(compute)) if i in finish]
    tl.mean_transfer_stall = sum(stalls) / len(stalls) if stalls else 0.0
    tl.idle_fraction = ((tl.total_latency - tl.total_compute) / tl.total_latency
                        if tl.total_latency > 0 else 0.0)
    return tl


def simulate_serial(compute, transfers, link: LinkModel, rate: float) -> Timeline:
    return _sim(compute, transfers, link, rate, False)


def simulate_pipelined(compute, transfers, link: LinkModel, rate: float) -> Timeline:
    return _sim(compute, transfers, link, rate, True)


def calibrated_step(fast_s: float, n_records: int, record_compute_s: float,
                    record_transfer_s: float) -> dict:
    """The reference's model of one GPU decode step with measured B200 rates:
    compute lane = the fast tier, then one item per streamed record; transfer
    lane = one item per record.  Rates are expressed as 1 unit/s so each
    item's amount is its measured duration (fast kernel time; slow-kernel time
    per record in the serial schedule; gather time per record)."""
    compute = [fast_s] + [record_compute_s] * n_records
    transfers = [(i + 1, record_transfer_s) for i in range(n_records)]
    link = LinkModel(bandwidth=1.0)
    pipe = simulate_pipelined(compute, transfers, link, 1.0)
    ser = simulate_serial(compute, transfers, link, 1.0)
    return {"pipelined_ms": pipe.total_latency * 1e3, "serial_ms": ser.total_latency * 1e3,
            "pipelined_idle_fraction": pipe.idle_fraction,
            "serial_idle_fraction": ser.idle_fraction,
            "pipelined_stall_ms": pipe.mean_transfer_stall * 1e3,
            "serial_stall_ms": ser.mean_transfer_stall * 1e3}


def run_sweep(tier, policy, spec, context_lengths=(), block_sizes=(), key_bits=(),
              value_bits=(), fetch_fractions=(), **kw) -> List[RunRecord]:
    """run_sweep (harness.cpp:173-208): deterministic grid order."""
    out = []
    for ctx in context_lengths or (spec.context_length,):
        for blk in block_sizes or (tier.block_size,):
            for kb in key_bits or (tier.key_bits,):
                for vb in value_bits or (tier.value_bits,):
                    for fr in fetch_fractions or (policy.fetch_fraction,):
                        t = replace(tier, block_size=blk, key_bits=kb, value_bits=vb)
                        p = replace(policy, fetch_fraction=fr)
                        out.append(run_benchmark(t, p, replace(spec, context_length=ctx), **kw))
    return out


def run_ablation(tier, policy, spec, **kw) -> List[RunRecord]:
    """run_ablation (harness.cpp:210-221): same order as the reference."""
    return [run_benchmark(tier, policy, spec, baseline=b, **kw) for b in ABLATION_ORDER]


def _fmt(v) -> str:
    return "%.10g" % v


REPORT_COLUMNS = ["method", "context_length", "block_size", "key_bits", "value_bits",
                  "fetch_fraction", "h2g_bytes", "traffic_reduction", "p95_latency",
                  "throughput", "oracle_error", "needle_recall", "pcie_bytes_measured",
                  "mean_latency"]


def _row(r: RunRecord) -> dict:
    s = r.summary
    recall = (r.needle_hits / len(r.latency_ms)) if (r.spec.kind == "needle" and r.latency_ms) \
        else None
    return dict(method=r.method, context_length=r.spec.context_length,
                block_size=r.tier.block_size, key_bits=r.tier.key_bits,
                value_bits=r.tier.value_bits, fetch_fraction=r.policy.fetch_fraction,
                h2g_bytes=s["total_h2g_bytes"], traffic_reduction=s["traffic_reduction"],
                p95_latency=s["p95_latency_ms"] / 1e3, throughput=s["tokens_per_second"],
                oracle_error=(sum(r.oracle_errors) / len(r.oracle_errors))
                if r.oracle_errors else 0.0,
                needle_recall=recall, pcie_bytes_measured=s["pcie_bytes_measured"],
                mean_latency=s["mean_latency_ms"] / 1e3)


def write_report(records: List[RunRecord], fmt: str = "csv") -> str:
    """write_report (harness.cpp:225-277).  The reference's `_model` latency
    columns carry measured seconds here (p95_latency, throughput); two
    measured columns are appended."""
    if not records:
        raise ValueError("write_report: no run records")
    rows = [_row(r) for r in records]
    if fmt == "json":
        return json.dumps(rows, indent=2) + "\n"
    lines = [",".join(REPORT_COLUMNS)]
    for d in rows:
        cells = []
        for c in REPORT_COLUMNS:
            v = d[c]
            cells.append("" if v is None else (_fmt(v) if isinstance(v, float) else str(v)))
        lines.append(",".join(cells))
    return "\n".join(lines) + "\n"


def write_step_records(r: RunRecord) -> str:
    """write_step_records (harness.cpp:279-289) with measured latency."""
    lines = ["step,latency,bytes_transferred,blocks_scored,blocks_fetched,eviction,"
             "oracle_error,pcie_bytes_measured"]
    for i in range(len(r.latency_ms)):
        err = r.oracle_errors[i] if r.oracle_errors else 0.0
        lines.append(f"{i},{_fmt(r.latency_ms[i] / 1e3)},{_fmt(r.step_bytes[i])},"
                     f"{r.blocks_scored[i]},{r.blocks_fetched[i]},{int(r.evictions[i])},"
                     f"{_fmt(err)},{r.pcie_bytes[i]}")
    return "\n".join(lines) + "\n"


def write_run_timelines(r: RunRecord) -> str:
    """write_run_timelines (harness.cpp:291-300): `step lane label start finish`
    (seconds), one line per event.  The events are the measured B200 kernels of
    each step; the PCIe-streaming slow-tier kernel is the transfer lane, every
    other kernel the compute lane."""
    out = []
    for i, tl in enumerate(r.timelines):
        for name, a, b in tl:
            lane = "transfer" if name in ("slow", "gather") else "compute"
            out.append(f"{i}\t{lane}\t{name}\t{_fmt(a * 1e-3)}\t{_fmt(b * 1e-3)}")
    return "\n".join(out) + ("\n" if out else "")


def emit_report(records: List[RunRecord], out_dir: str, fmt: str = "csv") -> None:
    """emit_report (harness.cpp:302-322): report.{csv,json} + steps-NNN.csv."""
    if not records:
        raise ValueError("emit_report: no run records")
    os.makedirs(out_dir, exist_ok=True)
    with open(os.path.join(out_dir, "report." + fmt), "w") as f:
        f.write(write_report(records, fmt))
    for i, r in enumerate(records):
        with open(os.path.join(out_dir, "steps-%03d.csv" % i), "w") as f:
            f.write(write_step_records(r))
