"""ctypes binding of the C ABI in include/ttkv_gpu.h (libttkv_gpu.so, sm_100a).

The library is built in-tree (``make lib`` / ``__graft_entry__.build()``).  There
is no CPU fallback: if the library or a CUDA device is missing, calls raise.
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "lib", "libttkv_gpu.so")

TTKV_OK, TTKV_ECONFIG, TTKV_ESEQUENCE, TTKV_ESHAPE = 0, 1, 2, 3
TTKV_EINTEGRITY, TTKV_EIO, TTKV_EERROR, TTKV_ECUDA, TTKV_EINVAL = 4, 5, 6, 7, 8
DTYPE_F32, DTYPE_F16 = 0, 1
SLOW_PINNED_HOST, SLOW_DEVICE = 0, 1


class TierConfigC(C.Structure):
    _fields_ = [("hbm_budget_bytes", C.c_uint64), ("d_k", C.c_uint64), ("d_v", C.c_uint64),
                ("bytes_full_precision", C.c_uint64), ("block_size", C.c_uint64),
                ("key_bits", C.c_uint32), ("value_bits", C.c_uint32),
                ("fetch_fraction", C.c_double), ("has_top_k_blocks", C.c_int32),
                ("top_k_blocks", C.c_uint64), ("hbm_bandwidth", C.c_double),
                ("pcie_bandwidth", C.c_double), ("transfer_latency", C.c_double),
                ("compute_rate", C.c_double)]


class SelectionPolicyC(C.Structure):
    _fields_ = [("has_top_k", C.c_int32), ("top_k", C.c_uint64), ("fetch_fraction", C.c_double)]


class OptionsC(C.Structure):
    _fields_ = [("device", C.c_int32), ("n_streams", C.c_uint32),
                ("heads_per_stream", C.c_uint32), ("group_select", C.c_uint32),
                ("reserve_tokens", C.c_uint64), ("slow_tier", C.c_uint32),
                ("copy_mode", C.c_uint32), ("literal_additive_merge", C.c_uint32),
                ("ring_bytes", C.c_uint32), ("serial_schedule", C.c_uint32),
                ("record_stream", C.c_uint32)]


class StepReportC(C.Structure):
    _fields_ = [("blocks_scored", C.c_uint64), ("blocks_fetched", C.c_uint64),
                ("bytes_transferred", C.c_double), ("fast_tokens", C.c_uint64),
                ("eviction_occurred", C.c_int32), ("union_blocks", C.c_uint64),
                ("pcie_bytes", C.c_uint64)]


class StateC(C.Structure):
    _fields_ = [(n, C.c_uint64) for n in (
        "appended", "fast_tokens", "slow_blocks", "l_fast", "record_bytes",
        "modeled_block_bytes", "n_streams", "heads_per_stream", "block_capacity", "launches",
        "payload_bytes", "graph_replays", "graph_captures", "spec_steps")]


class KernelTimesC(C.Structure):
    _fields_ = ([("ms_" + n, C.c_double) for n in
                 ("append", "score", "select", "fast", "slow", "combine", "evict")] +
                [("n_" + n, C.c_uint64) for n in
                 ("append", "score", "select", "fast", "slow", "combine", "evict")] +
                [("ms_gather", C.c_double), ("n_gather", C.c_uint64),
                 ("ms_step", C.c_double), ("n_step", C.c_uint64),
                 ("last_step_ms", C.c_double)])


# every symbol include/ttkv_gpu.h declares (checked by tests/test_abi.py)
EXPORTS = [
    "ttkv_gpu_create", "ttkv_gpu_destroy", "ttkv_gpu_last_error", "ttkv_last_error",
    "ttkv_abi_version", "ttkv_device_count", "ttkv_gpu_set_stream", "ttkv_gpu_get_stream",
    "ttkv_gpu_synchronize", "ttkv_gpu_prefill", "ttkv_gpu_prefill_synthetic",
    "ttkv_gpu_prefill_device",
    "ttkv_gpu_decode_step", "ttkv_gpu_decode_step_device", "ttkv_gpu_read_step_counters",
    "ttkv_gpu_state", "ttkv_gpu_read_fetched", "ttkv_gpu_read_selected", "ttkv_gpu_read_union",
    "ttkv_gpu_read_scores", "ttkv_gpu_read_block", "ttkv_gpu_serialize_block",
    "ttkv_gpu_dump_slow_tier", "ttkv_gpu_restore_slow_tier", "ttkv_gpu_read_fast", "ttkv_gpu_locate", "ttkv_gpu_set_timing",
    "ttkv_gpu_kernel_times", "ttkv_gpu_read_timeline", "ttkv_gpu_peer_gather_init",
    "ttkv_gpu_peer_gather_open", "ttkv_gpu_peer_gather_output", "ttkv_gpu_peer_gather_close",
    "ttkv_gpu_quantize_block",
    "ttkv_gpu_append", "ttkv_gpu_evict",
    "ttkv_gpu_eviction_pending", "ttkv_gpu_dequantize_block", "ttkv_gpu_score_blocks",
    "ttkv_gpu_select_top_k", "ttkv_fast_capacity",
    "ttkv_modeled_block_bytes", "ttkv_packed_bytes", "ttkv_resolve", "ttkv_validate_config",
    "ttkv_default_config", "ttkv_pci_bus_id", "ttkv_peer_probe",
]

_lib = None


def lib():
    """Load libttkv_gpu.so; raise loudly if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise RuntimeError(f"{LIB_PATH} missing: build it with `make lib` "
                           "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    vp, u32, u64, i32 = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
    P = C.POINTER
    sig = {
        "ttkv_gpu_create": (i32, [P(TierConfigC), P(SelectionPolicyC), P(OptionsC), P(vp)]),
        "ttkv_gpu_destroy": (None, [vp]),
        "ttkv_gpu_last_error": (C.c_char_p, [vp]),
        "ttkv_last_error": (C.c_char_p, []),
        "ttkv_abi_version": (i32, []),
        "ttkv_device_count": (i32, [P(i32)]),
        "ttkv_gpu_set_stream": (i32, [vp, vp]),
        "ttkv_gpu_get_stream": (vp, [vp]),
        "ttkv_gpu_synchronize": (i32, [vp]),
        "ttkv_gpu_prefill": (i32, [vp, vp, vp, u64, i32]),
        "ttkv_gpu_prefill_synthetic": (i32, [vp, u64, u64]),
        "ttkv_gpu_prefill_device": (i32, [vp, vp, vp, u64, i32]),
        "ttkv_gpu_decode_step": (i32, [vp, vp, vp, vp, i32, vp, P(StepReportC)]),
        "ttkv_gpu_decode_step_device": (i32, [vp, vp, vp, vp, i32, vp, P(StepReportC)]),
        "ttkv_gpu_read_step_counters": (i32, [vp, P(u64), P(u64)]),
        "ttkv_gpu_state": (i32, [vp, P(StateC)]),
        "ttkv_gpu_read_fetched": (i32, [vp, u32, u32, vp, u64, P(u64)]),
        "ttkv_gpu_read_selected": (i32, [vp, u32, u32, vp, u64, P(u64)]),
        "ttkv_gpu_read_union": (i32, [vp, u32, vp, vp, u64, P(u64)]),
        "ttkv_gpu_read_scores": (i32, [vp, u32, u32, vp, u64, P(u64)]),
        "ttkv_gpu_read_block": (i32, [vp, u32, u64, vp, vp, vp, vp, vp, P(u64)]),
        "ttkv_gpu_serialize_block": (i32, [vp, u32, u64, vp, u64, P(u64)]),
        "ttkv_gpu_dump_slow_tier": (i32, [vp, u32, C.c_char_p]),
        "ttkv_gpu_restore_slow_tier": (i32, [vp, P(C.c_char_p), u32]),
        "ttkv_gpu_read_fast": (i32, [vp, u32, vp, vp, u64, P(u64), P(u64)]),
        "ttkv_gpu_locate": (i32, [vp, u64, P(i32), P(u64)]),
        "ttkv_gpu_set_timing": (i32, [vp, i32]),
        "ttkv_gpu_kernel_times": (i32, [vp, P(KernelTimesC), i32]),
        "ttkv_gpu_read_timeline": (i32, [vp, vp, vp, vp, u64, P(u64)]),
        "ttkv_gpu_peer_gather_init": (i32, [vp, u32, u32, u64, vp, vp]),
        "ttkv_gpu_peer_gather_open": (i32, [vp, vp]),
        "ttkv_gpu_peer_gather_output": (i32, [vp, P(vp), P(i32)]),
        "ttkv_gpu_peer_gather_close": (i32, [vp]),
        "ttkv_gpu_quantize_block": (i32, [i32, vp, vp, u64, u32, u32, u32, u32, vp, vp, vp, vp,
                                          vp]),
        "ttkv_gpu_append": (i32, [vp, vp, vp, u64, i32]),
        "ttkv_gpu_evict": (i32, [vp, P(u64)]),
        "ttkv_gpu_eviction_pending": (i32, [vp, P(i32)]),
        "ttkv_gpu_dequantize_block": (i32, [i32, vp, vp, vp, vp, u64, u32, u32, u32, u32, vp,
                                            vp]),
        "ttkv_gpu_score_blocks": (i32, [i32, vp, vp, u64, u32, vp]),
        "ttkv_gpu_select_top_k": (i32, [i32, vp, vp, u64, u64, vp]),
        "ttkv_fast_capacity": (u64, [P(TierConfigC)]),
        "ttkv_modeled_block_bytes": (u64, [P(TierConfigC)]),
        "ttkv_packed_bytes": (u64, [u64, u32]),
        "ttkv_resolve": (u64, [P(SelectionPolicyC), u64]),
        "ttkv_validate_config": (i32, [P(TierConfigC)]),
        "ttkv_default_config": (None, [P(TierConfigC)]),
        "ttkv_pci_bus_id": (i32, [i32, C.c_char_p, i32]),
        "ttkv_peer_probe": (i32, [i32, C.c_char_p, P(i32)]),
    }
    for name, (res, args) in sig.items():
        f = getattr(L, name)
        f.restype = res
        f.argtypes = args
    _lib = L
    return L
