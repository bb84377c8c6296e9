"""Python mirror of the reference's tier-manager / engine API over the C ABI.

Names, argument meaning and error classes follow the reference
(/root/reference/proj/core/include/ttkv/):
  TierConfig      config.hpp:14-75        SelectionPolicy  relevance.hpp:19-24
  Engine          engine.hpp:36-49        DecodeStepReport engine.hpp:21-29
  errors          errors.hpp:8-41
``MultiStreamEngine`` is the batched form the B200 path is built around: S KV
streams (layers x KV heads x requests) in lockstep, G query heads each.
Everything runs in libttkv_gpu.so; there is no CPU fallback.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from . import _lib as L


# --- errors (errors.hpp:8-41) -------------------------------------------------
class Error(RuntimeError):
    pass


class ConfigError(Error):
    pass


class SequencingError(Error):
    pass


class ShapeError(Error):
    pass


class IntegrityError(Error):
    pass


class IoError(Error):
    pass


class CudaError(Error):
    pass


_ERR = {L.TTKV_ECONFIG: ConfigError, L.TTKV_ESEQUENCE: SequencingError,
        L.TTKV_ESHAPE: ShapeError, L.TTKV_EINTEGRITY: IntegrityError, L.TTKV_EIO: IoError,
        L.TTKV_EERROR: Error, L.TTKV_ECUDA: CudaError, L.TTKV_EINVAL: Error}


def _check(rc, h=None):
    if rc != L.TTKV_OK:
        lib = L.lib()
        msg = (lib.ttkv_gpu_last_error(h) if h else lib.ttkv_last_error()) or b""
        raise _ERR.get(rc, Error)(msg.decode(errors="replace"))


# --- config ------------------------------------------------------------------
@dataclass
class TierConfig:
    """config.hpp:14-41.  bytes_full_precision: 2 -> fp16 ring, 4 -> fp32 ring."""
    hbm_budget_bytes: int = 0
    d_k: int = 64
    d_v: int = 64
    bytes_full_precision: int = 2
    block_size: int = 128
    key_bits: int = 8
    value_bits: int = 4
    fetch_fraction: float = 0.45
    top_k_blocks: Optional[int] = None
    hbm_bandwidth: float = 2.0e12
    pcie_bandwidth: float = 3.2e10
    transfer_latency: float = 1.0e-5
    compute_rate: float = 4.0e11

    def d_kv(self):
        return self.d_k + self.d_v

    def block_bytes_full_precision(self):
        return self.block_size * self.d_kv() * self.bytes_full_precision

    def to_c(self) -> L.TierConfigC:
        return L.TierConfigC(self.hbm_budget_bytes, self.d_k, self.d_v,
                             self.bytes_full_precision, self.block_size, self.key_bits,
                             self.value_bits, self.fetch_fraction,
                             int(self.top_k_blocks is not None), self.top_k_blocks or 0,
                             self.hbm_bandwidth, self.pcie_bandwidth, self.transfer_latency,
                             self.compute_rate)

    def validate(self):
        c = self.to_c()
        _check(L.lib().ttkv_validate_config(C.byref(c)))


@dataclass
class SelectionPolicy:
    """relevance.hpp:19-24"""
    top_k: Optional[int] = None
    fetch_fraction: float = 0.45

    def to_c(self):
        return L.SelectionPolicyC(int(self.top_k is not None), self.top_k or 0,
                                  self.fetch_fraction)

    def resolve(self, block_count: int) -> int:
        c = self.to_c()
        k = L.lib().ttkv_resolve(C.byref(c), block_count)
        if k == 2 ** 64 - 1:
            _check(L.TTKV_ECONFIG)
        return k


def fast_capacity(cfg: TierConfig) -> int:
    """tier_store.cpp:36-44"""
    c = cfg.to_c()
    n = L.lib().ttkv_fast_capacity(C.byref(c))
    if n == 0:
        _check(L.TTKV_ECONFIG)
    return n


def modeled_block_bytes(cfg: TierConfig) -> int:
    c = cfg.to_c()
    return L.lib().ttkv_modeled_block_bytes(C.byref(c))


def compressed_bytes_per_token(cfg: TierConfig) -> float:
    return modeled_block_bytes(cfg) / cfg.block_size


def packed_bytes(count: int, bits: int) -> int:
    return L.lib().ttkv_packed_bytes(count, bits)


def device_count() -> int:
    n = C.c_int(0)
    rc = L.lib().ttkv_device_count(C.byref(n))
    return n.value if rc == 0 else 0


@dataclass
class DecodeStepReport:
    """engine.hpp:21-29 (+ measured transfer counters)."""
    output: np.ndarray
    blocks_scored: int = 0
    blocks_fetched: int = 0
    fetched_blocks: List[np.ndarray] = field(default_factory=list)
    bytes_transferred: float = 0.0
    eviction_occurred: bool = False
    fast_tokens: int = 0
    union_blocks: int = 0
    pcie_bytes: int = 0


def _f32(x):
    return np.ascontiguousarray(x, dtype=np.float32)


def _kv(x):
    x = np.ascontiguousarray(x)
    if x.dtype == np.float16:
        return x, L.DTYPE_F16
    return np.ascontiguousarray(x, dtype=np.float32), L.DTYPE_F32


def _ptr(a):
    return a.ctypes.data_as(C.c_void_p)


class _AddrCache:
    """Data addresses of the last few arrays passed to the per-token call
    (a.ctypes.data costs ~1.3-2.4 us per array).  Each entry holds its array,
    so its id cannot be reused by another object and its buffer cannot be
    resized (ndarray.resize refuses while another reference exists)."""

    def __init__(self, size=16):
        self._d = {}
        self._size = size

    def __call__(self, a):
        e = self._d.get(id(a))
        if e is not None and e[0] is a:
            return e[1]
        if len(self._d) >= self._size:
            self._d.pop(next(iter(self._d)))
        addr = a.ctypes.data
        self._d[id(a)] = (a, addr)
        return addr


class MultiStreamEngine:
    """S lockstep KV streams x G query heads on one B200 (include/ttkv_gpu.h)."""

    def __init__(self, config: TierConfig, policy: SelectionPolicy = None, n_streams: int = 1,
                 heads_per_stream: int = 1, group_select: bool = False, device: int = 0,
                 reserve_tokens: int = 0, slow_tier: int = L.SLOW_PINNED_HOST,
                 copy_mode: int = 0, literal_additive_merge: bool = False,
                 ring_bytes: int = 0, serial_schedule: bool = False, record_stream: int = 0):
        self.config = config
        self.policy = policy or SelectionPolicy(config.top_k_blocks, config.fetch_fraction)
        self.S, self.G = n_streams, heads_per_stream
        self.device = device
        self._lib = L.lib()
        self._rep = L.StepReportC()  # reused by decode_step (its fields are copied out)
        self._rep_ref = C.byref(self._rep)
        self._addr = _AddrCache()
        self._c_cfg = config.to_c()
        self._c_pol = self.policy.to_c()
        self._c_opt = L.OptionsC(device, n_streams, heads_per_stream, int(group_select),
                                 reserve_tokens, slow_tier, copy_mode,
                                 int(literal_additive_merge), ring_bytes,
                                 int(serial_schedule), record_stream)
        h = C.c_void_p()
        _check(self._lib.ttkv_gpu_create(C.byref(self._c_cfg), C.byref(self._c_pol),
                                         C.byref(self._c_opt), C.byref(h)))
        self._h = h

    # lifecycle --------------------------------------------------------------
    def close(self):
        if getattr(self, "_h", None):
            self._lib.ttkv_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def handle(self):
        return self._h

    # hot path ----------------------------------------------------------------
    def prefill(self, keys, values):
        """keys [S, n, d_k], values [S, n, d_v] (float32 or float16)."""
        k, dt = _kv(keys)
        v, dt2 = _kv(values)
        if dt != dt2:
            raise ShapeError("prefill: keys and values must share a dtype")
        if k.ndim == 2:
            k, v = k[None], v[None]
        if k.shape[0] != self.S or k.shape[2] != self.config.d_k or v.shape[2] != self.config.d_v \
                or v.shape[:2] != k.shape[:2]:
            raise ShapeError("prefill: key/value dimension mismatch")
        _check(self._lib.ttkv_gpu_prefill(self._h, _ptr(k), _ptr(v), k.shape[1], dt), self._h)

    def prefill_device(self, k_ptr: int, v_ptr: int, n_tokens: int, dtype: int = L.DTYPE_F16):
        """Prefill from device rows [S][n][d] (e.g. torch tensors' data_ptr())."""
        _check(self._lib.ttkv_gpu_prefill_device(self._h, C.c_void_p(k_ptr), C.c_void_p(v_ptr),
                                                 n_tokens, dtype), self._h)

    def prefill_synthetic(self, n_tokens: int, seed: int = 0):
        _check(self._lib.ttkv_gpu_prefill_synthetic(self._h, n_tokens, seed), self._h)

    def decode_step(self, query, key, value, fetched=False, out=None) -> DecodeStepReport:
        """query [S, G, d_k], key [S, d_k], value [S, d_v] -> output [S, G, d_v].
        `out` (optional): a C-contiguous float64 [S, G, d_v] array the output is
        written to.  Page-locked inputs / `out` (e.g. numpy views of
        torch.empty(..., pin_memory=True)) are read and written by the step's
        kernels in place (device mapping); pageable ones go through the
        handle's page-locked staging buffers."""
        q = _f32(query)  # the caller's array itself when already f32 and contiguous
        k, dt = _kv(key)
        v, _ = _kv(value)
        if v.dtype != k.dtype:
            v = v.astype(k.dtype)
        if q.size != self.S * self.G * self.config.d_k:
            raise ShapeError("decode_step: query dimension mismatch")
        if k.size != self.S * self.config.d_k or v.size != self.S * self.config.d_v:
            raise ShapeError("append_token: key/value dimension mismatch")
        shape = (self.S, self.G, self.config.d_v)
        out_given = out is not None
        if out is None:
            out = np.empty(shape, np.float64)  # fully written by the call
        elif out.dtype != np.float64 or out.shape != shape or not out.flags.c_contiguous:
            raise ShapeError("decode_step: out must be a C-contiguous float64 [S, G, d_v] array")
        rep = self._rep
        # cached addresses for the caller's own arrays (reused step after
        # step); converted temporaries are looked up directly
        ad = self._addr
        aq = ad(q) if q is query else q.ctypes.data
        ak = ad(k) if k is key else k.ctypes.data
        av = ad(v) if v is value else v.ctypes.data
        ao = ad(out) if out_given else out.ctypes.data
        _check(self._lib.ttkv_gpu_decode_step(self._h, aq, ak, av, dt, ao, self._rep_ref),
               self._h)
        # positional: the per-token path (keyword arguments cost ~0.6 us more)
        r = DecodeStepReport(out, rep.blocks_scored, rep.blocks_fetched, [],
                             rep.bytes_transferred, bool(rep.eviction_occurred), rep.fast_tokens,
                             rep.union_blocks, rep.pcie_bytes)
        if fetched:
            r.fetched_blocks = [[self.read_fetched(s, g) for g in range(self.G)]
                                for s in range(self.S)]
        return r

    def decode_step_device(self, q_ptr: int, k_ptr: int, v_ptr: int, out_ptr: int,
                           dtype: int = L.DTYPE_F16):
        """Device pointers (ints), enqueued on the handle's stream."""
        rep = L.StepReportC()
        _check(self._lib.ttkv_gpu_decode_step_device(self._h, C.c_void_p(q_ptr),
                                                     C.c_void_p(k_ptr), C.c_void_p(v_ptr), dtype,
                                                     C.c_void_p(out_ptr), C.byref(rep)), self._h)
        return rep

    def set_stream(self, stream_ptr: int):
        _check(self._lib.ttkv_gpu_set_stream(self._h, C.c_void_p(stream_ptr)), self._h)

    def synchronize(self):
        _check(self._lib.ttkv_gpu_synchronize(self._h), self._h)

    def step_counters(self):
        u, p = C.c_uint64(), C.c_uint64()
        _check(self._lib.ttkv_gpu_read_step_counters(self._h, C.byref(u), C.byref(p)), self._h)
        return u.value, p.value

    # state / cold path ---------------------------------------------------------
    def state(self) -> dict:
        st = L.StateC()
        _check(self._lib.ttkv_gpu_state(self._h, C.byref(st)), self._h)
        return {n: getattr(st, n) for n, _ in L.StateC._fields_}

    def read_fetched(self, stream: int, head: int = 0) -> np.ndarray:
        n = C.c_uint64()
        _check(self._lib.ttkv_gpu_read_fetched(self._h, stream, head, None, 0, C.byref(n)),
               self._h)
        out = np.zeros(max(1, n.value), np.uint64)
        _check(self._lib.ttkv_gpu_read_fetched(self._h, stream, head, _ptr(out), n.value,
                                               C.byref(n)), self._h)
        return out[:n.value]

    def read_selected(self, stream: int, head: int = 0) -> np.ndarray:
        """The block ids the last step's slow kernel streamed for (stream,
        head), ascending (the GPU's own top-k set)."""
        n = C.c_uint64()
        _check(self._lib.ttkv_gpu_read_selected(self._h, stream, head, None, 0, C.byref(n)),
               self._h)
        out = np.zeros(max(1, n.value), np.uint32)
        _check(self._lib.ttkv_gpu_read_selected(self._h, stream, head, _ptr(out), n.value,
                                                C.byref(n)), self._h)
        return out[:n.value]

    def read_union(self, stream: int):
        """(ids, head_masks) of the last step's per-stream union, ascending."""
        n = C.c_uint64()
        _check(self._lib.ttkv_gpu_read_union(self._h, stream, None, None, 0, C.byref(n)), self._h)
        ids = np.zeros(max(1, n.value), np.uint32)
        masks = np.zeros(max(1, n.value), np.uint32)
        _check(self._lib.ttkv_gpu_read_union(self._h, stream, _ptr(ids), _ptr(masks), n.value,
                                             C.byref(n)), self._h)
        return ids[:n.value], masks[:n.value]

    def read_scores(self, stream: int, head: int = 0) -> np.ndarray:
        """The last step's fp64 block scores for (stream, head)."""
        n = C.c_uint64()
        _check(self._lib.ttkv_gpu_read_scores(self._h, stream, head, None, 0, C.byref(n)), self._h)
        out = np.zeros(max(1, n.value), np.float64)
        _check(self._lib.ttkv_gpu_read_scores(self._h, stream, head, _ptr(out), n.value,
                                              C.byref(n)), self._h)
        return out[:n.value]

    def read_block(self, stream: int, block_id: int) -> dict:
        cfg = self.config
        B = cfg.block_size
        pk = np.zeros(max(1, packed_bytes(B * cfg.d_k, cfg.key_bits)), np.uint8)
        pv = np.zeros(max(1, packed_bytes(B * cfg.d_v, cfg.value_bits)), np.uint8)
        kp = np.zeros(2 * cfg.d_k, np.float32)
        vp = np.zeros(2 * cfg.d_v, np.float32)
        cen = np.zeros(cfg.d_k, np.float32)
        first = C.c_uint64()
        _check(self._lib.ttkv_gpu_read_block(self._h, stream, block_id, _ptr(pk), _ptr(pv),
                                             _ptr(kp), _ptr(vp), _ptr(cen), C.byref(first)),
               self._h)
        return dict(packed_keys=pk, packed_values=pv, key_params=kp, value_params=vp,
                    key_centroid=cen, first_position=first.value)

    def serialize_block(self, stream: int, block_id: int) -> bytes:
        n = C.c_uint64()
        _check(self._lib.ttkv_gpu_serialize_block(self._h, stream, block_id, None, 0,
                                                  C.byref(n)), self._h)
        buf = (C.c_uint8 * n.value)()
        _check(self._lib.ttkv_gpu_serialize_block(self._h, stream, block_id, buf, n.value,
                                                  C.byref(n)), self._h)
        return bytes(buf)

    def dump_slow_tier(self, stream: int, path: str):
        _check(self._lib.ttkv_gpu_dump_slow_tier(self._h, stream, str(path).encode()), self._h)

    def restore_slow_tier(self, paths):
        """Rebuild this (fresh) handle's slow tier from one TTKVTIER file per
        stream (load_slow_tier, quantizer.cpp:344-365)."""
        arr = (C.c_char_p * len(paths))(*[str(p).encode() for p in paths])
        _check(self._lib.ttkv_gpu_restore_slow_tier(self._h, arr, len(paths)), self._h)

    def append(self, keys, values):
        """append_token for n tokens of every stream: keys [S, n, d_k]."""
        k, dt = _kv(keys)
        v, _ = _kv(values)
        if v.dtype != k.dtype:
            v = v.astype(k.dtype)
        if k.ndim == 2:
            k, v = k[:, None], v[:, None]
        _check(self._lib.ttkv_gpu_append(self._h, _ptr(k), _ptr(v), k.shape[1], dt), self._h)

    def checkpoint(self, directory):
        """Checkpoint every stream: its slow tier in the reference's TTKVTIER
        format (dump_slow_tier, byte-identical) plus the fast-tier rows."""
        os.makedirs(directory, exist_ok=True)
        ks, vs, first = [], [], 0
        for s in range(self.S):
            self.dump_slow_tier(s, os.path.join(directory, f"stream_{s:05d}.ttkvtier"))
            k, v, first = self.read_fast(s)
            ks.append(k)
            vs.append(v)
        np.savez(os.path.join(directory, "fast_tier.npz"), keys=np.stack(ks),
                 values=np.stack(vs), first_position=first)

    def restore(self, directory):
        """Resume a fresh handle from checkpoint(): slow tier, then fast tier."""
        self.restore_slow_tier([os.path.join(directory, f"stream_{s:05d}.ttkvtier")
                                for s in range(self.S)])
        ft = np.load(os.path.join(directory, "fast_tier.npz"))
        if int(ft["first_position"]) != self.state()["appended"]:
            raise IntegrityError("restore: fast tier does not continue the slow tier")
        if ft["keys"].shape[1]:
            self.append(ft["keys"], ft["values"])

    def read_fast(self, stream: int):
        n, first = C.c_uint64(), C.c_uint64()
        _check(self._lib.ttkv_gpu_read_fast(self._h, stream, None, None, 0, C.byref(n),
                                            C.byref(first)), self._h)
        k = np.zeros((max(1, n.value), self.config.d_k), np.float32)
        v = np.zeros((max(1, n.value), self.config.d_v), np.float32)
        _check(self._lib.ttkv_gpu_read_fast(self._h, stream, _ptr(k), _ptr(v), n.value,
                                            C.byref(n), C.byref(first)), self._h)
        return k[:n.value], v[:n.value], first.value

    def locate(self, position: int):
        w, b = C.c_int(), C.c_uint64()
        _check(self._lib.ttkv_gpu_locate(self._h, position, C.byref(w), C.byref(b)), self._h)
        return ("fast", "slow", "absent")[w.value], b.value

    # measurement ---------------------------------------------------------------
    def set_timing(self, on: bool):
        _check(self._lib.ttkv_gpu_set_timing(self._h, int(on)), self._h)

    KERNEL_NAMES = ("append", "score", "select", "fast", "slow", "combine", "evict", "gather")

    def timeline(self):
        """Kernels of the last timed step: [(name, start_ms, end_ms)] from the
        step's start (ttkv_gpu_read_timeline)."""
        n = C.c_uint64()
        _check(self._lib.ttkv_gpu_read_timeline(self._h, None, None, None, 0, C.byref(n)),
               self._h)
        k = np.zeros(max(1, n.value), np.uint32)
        a = np.zeros(max(1, n.value), np.float64)
        b = np.zeros(max(1, n.value), np.float64)
        _check(self._lib.ttkv_gpu_read_timeline(self._h, _ptr(k), _ptr(a), _ptr(b), n.value,
                                                C.byref(n)), self._h)
        return [(self.KERNEL_NAMES[int(k[i])], float(a[i]), float(b[i])) for i in range(n.value)]

    def kernel_times(self, reset=False) -> dict:
        t = L.KernelTimesC()
        _check(self._lib.ttkv_gpu_kernel_times(self._h, C.byref(t), int(reset)), self._h)
        return {n: getattr(t, n) for n, _ in L.KernelTimesC._fields_}


class Engine:
    """Single-stream drop-in for ttkv::Engine (engine.hpp:36-49): one KV
    stream, one query per step, reference report semantics."""

    def __init__(self, config: TierConfig, policy: SelectionPolicy = None, device: int = 0,
                 reserve_tokens: int = 0, ring_bytes: int = 4):
        # The reference stores float32 tokens whatever bytes_full_precision
        # says (kv_types.hpp:14-15), so the single-stream drop-in defaults to
        # an fp32 ring (fp64 accumulation); ring_bytes=2 selects fp16.
        self._m = MultiStreamEngine(config, policy, 1, 1, device=device,
                                    reserve_tokens=reserve_tokens, ring_bytes=ring_bytes)
        self.config = config
        self.policy = self._m.policy

    def prefill(self, keys, values):
        self._m.prefill(_f32(keys)[None] if np.asarray(keys).dtype != np.float16 else keys[None],
                        _f32(values)[None] if np.asarray(values).dtype != np.float16 else values[None])

    def decode_step(self, query, key, value) -> DecodeStepReport:
        if np.asarray(query).size != self.config.d_k:
            raise ShapeError("decode_step: query dimension mismatch")
        r = self._m.decode_step(_f32(query).reshape(1, 1, -1), np.asarray(key).reshape(1, -1),
                                np.asarray(value).reshape(1, -1))
        r.output = r.output.reshape(-1)
        r.fetched_blocks = self._m.read_fetched(0, 0)
        return r

    @property
    def store(self):
        return self._m

    def close(self):
        self._m.close()
