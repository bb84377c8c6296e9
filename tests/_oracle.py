"""ctypes bindings for the TEST-ONLY checkers under oracle/.

oracle/_build/libttkv_oracle.so  -- C restatement (oracle/ttkv_oracle.c)
oracle/_ref/libttkv_ref.so       -- unmodified reference core + oracle/ref_shim.cpp

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg import this.
"""
import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ORACLE_SO = os.path.join(ROOT, "oracle", "_build", "libttkv_oracle.so")
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libttkv_ref.so")

_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_u8p = np.ctypeslib.ndpointer(np.uint8, flags="C_CONTIGUOUS")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
sz = C.c_size_t


class TkoConfig(C.Structure):
    _fields_ = [("d_k", sz), ("d_v", sz), ("block_size", sz), ("l_fast", sz),
                ("key_bits", C.c_uint), ("value_bits", C.c_uint),
                ("has_top_k", C.c_int), ("top_k", sz), ("fetch_fraction", C.c_double)]


_oracle = None
_ref = None


def oracle():
    global _oracle
    if _oracle is None:
        if not os.path.exists(ORACLE_SO):
            raise RuntimeError("oracle not built: run `make -C oracle` or __graft_entry__.build()")
        L = C.CDLL(ORACLE_SO)
        L.tko_fast_capacity.restype = sz
        L.tko_fast_capacity.argtypes = [sz, sz, sz, sz]
        L.tko_packed_bytes.restype = sz
        L.tko_packed_bytes.argtypes = [sz, C.c_uint]
        L.tko_modeled_block_bytes.restype = sz
        L.tko_modeled_block_bytes.argtypes = [sz, sz, sz, C.c_uint, C.c_uint]
        L.tko_quantize_tensor.argtypes = [_f32p, sz, sz, C.c_uint, _f32p, _u8p]
        L.tko_dequantize_tensor.argtypes = [_u8p, sz, sz, C.c_uint, _f32p, _f32p]
        L.tko_centroid.argtypes = [_f32p, sz, sz, _f32p]
        L.tko_score_block.restype = C.c_double
        L.tko_score_block.argtypes = [_f32p, _f32p, sz]
        L.tko_resolve.restype = sz
        L.tko_resolve.argtypes = [C.c_int, sz, C.c_double, sz]
        L.tko_select_top_k.argtypes = [_f64p, C.c_void_p, sz, sz, _u64p]
        L.tko_engine_create.restype = C.c_void_p
        L.tko_engine_create.argtypes = [C.POINTER(TkoConfig)]
        L.tko_engine_destroy.argtypes = [C.c_void_p]
        L.tko_engine_prefill.argtypes = [C.c_void_p, _f32p, _f32p, sz]
        L.tko_engine_decode_step.argtypes = [C.c_void_p, _f32p, sz, C.c_int, _f32p, _f32p,
                                             _f64p, _u64p, sz, _u64p, C.POINTER(sz),
                                             C.POINTER(C.c_double), C.POINTER(sz),
                                             C.POINTER(C.c_int)]
        L.tko_engine_slow_blocks.restype = sz
        L.tko_engine_slow_blocks.argtypes = [C.c_void_p]
        L.tko_engine_fast_tokens.restype = sz
        L.tko_engine_fast_tokens.argtypes = [C.c_void_p]
        L.tko_engine_serialize_block.restype = sz
        L.tko_engine_serialize_block.argtypes = [C.c_void_p, sz, C.c_void_p]
        L.tko_engine_centroid.restype = C.POINTER(C.c_float)
        L.tko_engine_centroid.argtypes = [C.c_void_p, sz]
        L.tko_dense_attention.argtypes = [_f32p, sz, _f32p, _f32p, sz, sz, _f64p]
        L.tko_relative_error.restype = C.c_double
        L.tko_relative_error.argtypes = [_f64p, _f64p, sz]
        L.tko_generate_workload.argtypes = [C.c_int, sz, sz, sz, sz, C.c_uint64, sz, C.c_double,
                                            _f32p, _f32p, _f32p, _f32p, _f32p, C.c_void_p]
        _oracle = L
    return _oracle


def ref_available():
    return os.path.exists(REF_SO)


def ref():
    global _ref
    if _ref is None:
        L = C.CDLL(REF_SO)
        u32, u64 = C.c_uint32, C.c_uint64
        L.ref_last_error.restype = C.c_char_p
        L.ref_engine_create.restype = C.c_void_p
        L.ref_engine_create.argtypes = [u64, u32, u32, u32, u32, u32, u32, C.c_int, u64, C.c_double,
                                        C.c_int]
        L.ref_engine_destroy.argtypes = [C.c_void_p]
        L.ref_engine_prefill.argtypes = [C.c_void_p, _f32p, _f32p, u64]
        L.ref_engine_decode_step.argtypes = [C.c_void_p, _f32p, _f32p, _f32p, _f64p, _u64p, u64,
                                             C.POINTER(u64), C.POINTER(u64),
                                             C.POINTER(C.c_double), C.POINTER(C.c_int)]
        L.ref_engine_slow_blocks.restype = u64
        L.ref_engine_slow_blocks.argtypes = [C.c_void_p]
        L.ref_engine_fast_tokens.restype = u64
        L.ref_engine_fast_tokens.argtypes = [C.c_void_p]
        L.ref_engine_l_fast.restype = u64
        L.ref_engine_l_fast.argtypes = [C.c_void_p]
        L.ref_engine_serialize_block.restype = u64
        L.ref_engine_serialize_block.argtypes = [C.c_void_p, u64, C.c_void_p, u64]
        L.ref_quantize_serialize.restype = u64
        L.ref_quantize_serialize.argtypes = [_f32p, _f32p, u64, u32, u32, u32, u32, u64, u64,
                                             C.c_void_p, u64]
        L.ref_score_block.restype = C.c_double
        L.ref_score_block.argtypes = [_f32p, _f32p, u64]
        L.ref_select_top_k.restype = u64
        L.ref_select_top_k.argtypes = [_f64p, _u64p, u64, C.c_int, u64, C.c_double, _u64p]
        L.ref_fast_capacity.restype = u64
        L.ref_fast_capacity.argtypes = [u64, u32, u32, u32, u32]
        L.ref_modeled_block_bytes.restype = u64
        L.ref_modeled_block_bytes.argtypes = [u32, u32, u32, u32, u32]
        L.ref_generate_workload.argtypes = [C.c_int, u64, u64, u32, u32, u64, u64, C.c_double,
                                            _f32p, _f32p, _f32p, _f32p, _f32p]
        L.ref_dense_attention.argtypes = [_f32p, u32, _f32p, _f32p, u64, u32, _f64p]
        L.ref_traffic_reduction.restype = C.c_double
        L.ref_traffic_reduction.argtypes = [C.POINTER(u64)]
        L.ref_bench_decode.argtypes = [u32, u32, u64, u32, u32, u64, u32, u32, u32, u32,
                                       C.c_double, u64, _f64p, C.POINTER(C.c_double)]
        _ref = L
    return _ref


# ---------------------------------------------------------------------------
# Convenience wrappers
# ---------------------------------------------------------------------------

def packed_bytes(count, bits):
    return oracle().tko_packed_bytes(count, bits)


def quantize_tensor(data, bits):
    data = np.ascontiguousarray(data, np.float32)
    rows, dim = data.shape
    params = np.zeros(2 * dim, np.float32)
    packed = np.zeros(max(1, packed_bytes(rows * dim, bits)), np.uint8)
    oracle().tko_quantize_tensor(data.reshape(-1), rows, dim, bits, params, packed)
    return params, packed[:packed_bytes(rows * dim, bits)]


def dequantize_tensor(packed, rows, dim, bits, params):
    out = np.zeros(rows * dim, np.float32)
    oracle().tko_dequantize_tensor(np.ascontiguousarray(packed, np.uint8), rows, dim, bits,
                                   np.ascontiguousarray(params, np.float32), out)
    return out.reshape(rows, dim)


def generate_workload(ctx, T, d_k, d_v, seed, needle=False, needle_pos=2, strength=3.0,
                      use_ref=False):
    pk = np.zeros((max(ctx, 1), d_k), np.float32)
    pv = np.zeros((max(ctx, 1), d_v), np.float32)
    dk = np.zeros((max(T, 1), d_k), np.float32)
    dv = np.zeros((max(T, 1), d_v), np.float32)
    dq = np.zeros((max(T, 1), d_k), np.float32)
    if use_ref:
        rc = ref().ref_generate_workload(int(needle), ctx, T, d_k, d_v, seed, needle_pos, strength,
                                         pk.reshape(-1), pv.reshape(-1), dk.reshape(-1),
                                         dv.reshape(-1), dq.reshape(-1))
    else:
        rc = oracle().tko_generate_workload(int(needle), ctx, T, d_k, d_v, seed, needle_pos,
                                            strength, pk.reshape(-1), pv.reshape(-1),
                                            dk.reshape(-1), dv.reshape(-1), dq.reshape(-1), None)
    assert rc == 0
    return pk[:ctx], pv[:ctx], dk[:T], dv[:T], dq[:T]


class OracleEngine:
    """One KV stream shared by G query heads (oracle/ttkv_oracle.c)."""

    def __init__(self, d_k, d_v, block_size, l_fast, key_bits=8, value_bits=4,
                 top_k=None, fetch_fraction=0.45):
        self.cfg = TkoConfig(d_k, d_v, block_size, l_fast, key_bits, value_bits,
                             int(top_k is not None), top_k or 0, fetch_fraction)
        self.h = oracle().tko_engine_create(C.byref(self.cfg))
        assert self.h, "invalid oracle config"
        self.d_k, self.d_v = d_k, d_v

    def __del__(self):
        if getattr(self, "h", None):
            oracle().tko_engine_destroy(self.h)
            self.h = None

    def prefill(self, keys, values):
        keys = np.ascontiguousarray(keys, np.float32)
        values = np.ascontiguousarray(values, np.float32)
        oracle().tko_engine_prefill(self.h, keys.reshape(-1), values.reshape(-1), keys.shape[0])

    def decode_step(self, q, key, value, mode=0):
        q = np.ascontiguousarray(q, np.float32).reshape(-1, self.d_k)
        G = q.shape[0]
        cap = max(1, self.slow_blocks())
        out = np.zeros(G * self.d_v, np.float64)
        fetched = np.zeros(G * cap, np.uint64)
        nf = np.zeros(G, np.uint64)
        ns, ub, ev = sz(), sz(), C.c_int()
        by = C.c_double()
        rc = oracle().tko_engine_decode_step(
            self.h, q.reshape(-1), G, mode, np.ascontiguousarray(key, np.float32).reshape(-1),
            np.ascontiguousarray(value, np.float32).reshape(-1), out, fetched, cap, nf,
            C.byref(ns), C.byref(by), C.byref(ub), C.byref(ev))
        assert rc == 0
        fetched = fetched.reshape(G, cap)
        return dict(output=out.reshape(G, self.d_v),
                    fetched=[fetched[g, :int(nf[g])].copy() for g in range(G)],
                    blocks_scored=ns.value, bytes_transferred=by.value,
                    union_blocks=ub.value, eviction_occurred=bool(ev.value))

    def slow_blocks(self):
        return oracle().tko_engine_slow_blocks(self.h)

    def fast_tokens(self):
        return oracle().tko_engine_fast_tokens(self.h)

    def serialize_block(self, i):
        n = oracle().tko_engine_serialize_block(self.h, i, None)
        buf = (C.c_uint8 * n)()
        oracle().tko_engine_serialize_block(self.h, i, buf)
        return bytes(buf)

    def centroid(self, i):
        p = oracle().tko_engine_centroid(self.h, i)
        return np.ctypeslib.as_array(p, shape=(self.d_k,)).copy()


class RefEngine:
    """The unmodified reference ttkv::Engine (oracle/_ref)."""

    def __init__(self, budget, d_k, d_v, block_size, key_bits=8, value_bits=4, bytes_fp=2,
                 top_k=None, fetch_fraction=0.45, literal_merge=False):
        self.h = ref().ref_engine_create(budget, d_k, d_v, bytes_fp, block_size, key_bits,
                                         value_bits, int(top_k is not None), top_k or 0,
                                         fetch_fraction, int(literal_merge))
        if not self.h:
            raise ValueError(ref().ref_last_error().decode())
        self.d_k, self.d_v = d_k, d_v

    def __del__(self):
        if getattr(self, "h", None):
            ref().ref_engine_destroy(self.h)
            self.h = None

    def prefill(self, keys, values):
        keys = np.ascontiguousarray(keys, np.float32)
        values = np.ascontiguousarray(values, np.float32)
        assert ref().ref_engine_prefill(self.h, keys.reshape(-1), values.reshape(-1),
                                        keys.shape[0]) == 0

    def decode_step(self, q, key, value):
        cap = max(1, self.slow_blocks())
        out = np.zeros(self.d_v, np.float64)
        fetched = np.zeros(cap, np.uint64)
        nf, ns = C.c_uint64(), C.c_uint64()
        by, ev = C.c_double(), C.c_int()
        rc = ref().ref_engine_decode_step(
            self.h, np.ascontiguousarray(q, np.float32), np.ascontiguousarray(key, np.float32),
            np.ascontiguousarray(value, np.float32), out, fetched, cap, C.byref(nf),
            C.byref(ns), C.byref(by), C.byref(ev))
        assert rc == 0, ref().ref_last_error()
        return dict(output=out, fetched=fetched[:nf.value].copy(), blocks_scored=ns.value,
                    bytes_transferred=by.value, eviction_occurred=bool(ev.value))

    def slow_blocks(self):
        return ref().ref_engine_slow_blocks(self.h)

    def fast_tokens(self):
        return ref().ref_engine_fast_tokens(self.h)

    def l_fast(self):
        return ref().ref_engine_l_fast(self.h)

    def serialize_block(self, i):
        n = ref().ref_engine_serialize_block(self.h, i, None, 0)
        buf = (C.c_uint8 * n)()
        ref().ref_engine_serialize_block(self.h, i, buf, n)
        return bytes(buf)


def fp16_round(x):
    """Round to fp16-representable float32 values."""
    return np.asarray(x, np.float32).astype(np.float16).astype(np.float32)
