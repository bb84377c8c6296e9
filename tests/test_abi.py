"""C-ABI boundary checks that run without a GPU: the library loads, exports
every entry point include/ttkv_gpu.h declares, host-only helpers follow the
reference semantics, and device calls fail loudly (no CPU fallback)."""
import ctypes as C
import os
import re

import pytest

import paper_2604_19769_b200 as T
from paper_2604_19769_b200 import _lib as L

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    txt = open(os.path.join(ROOT, "include", "ttkv_gpu.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ttkv_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_declared_symbol():
    lib = L.lib()
    declared = header_functions()
    assert len(declared) >= 25
    for name in declared:
        assert hasattr(lib, name), name
    assert sorted(L.EXPORTS) == declared


def test_library_is_sm100a():
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {L.LIB_PATH} 2>&1").read()
    assert "sm_100a" in out


def test_abi_version():
    assert L.lib().ttkv_abi_version() == 1


def test_host_helpers_follow_reference():
    cfg = T.TierConfig(hbm_budget_bytes=1048576, d_k=128, d_v=128, bytes_full_precision=2)
    assert T.fast_capacity(cfg) == 2048                     # test_tier_store.cpp:38
    cfg.hbm_budget_bytes = 1048575
    assert T.fast_capacity(cfg) == 1920                     # :42
    cfg.hbm_budget_bytes = cfg.block_bytes_full_precision() - 1
    with pytest.raises(T.ConfigError):
        T.fast_capacity(cfg)
    c = T.TierConfig(d_k=128, d_v=128)
    assert T.modeled_block_bytes(c) == 25600                # test_quantizer.cpp:137
    assert T.compressed_bytes_per_token(c) == 200.0
    c.key_bits = c.value_bits = 16
    assert T.modeled_block_bytes(c) == 65536
    assert T.SelectionPolicy(None, 0.45).resolve(10) == 5   # test_relevance.cpp:8-20
    assert T.SelectionPolicy(None, 0.45).resolve(0) == 0
    assert T.SelectionPolicy(5).resolve(3) == 3
    assert T.SelectionPolicy(5).resolve(20) == 5
    with pytest.raises(T.ConfigError):
        T.SelectionPolicy(None, 1.5).resolve(3)


@pytest.mark.parametrize("field,value,msg", [
    ("d_k", 0, "d_k and d_v must be positive"),
    ("block_size", 0, "block_size must be positive"),
    ("key_bits", 9, "bit widths must be in [2,8] or 16"),
    ("value_bits", 16, "key_bits must be >= value_bits"),
    ("hbm_budget_bytes", 10, "HBM budget smaller than one full-precision block"),
    ("fetch_fraction", 0.0, "fetch_fraction must be in (0, 1]"),
    ("pcie_bandwidth", 0.0, "bandwidths and compute_rate must be positive"),
    ("transfer_latency", -1.0, "transfer_latency must be non-negative"),
])
def test_validate_messages(field, value, msg):
    cfg = T.TierConfig(hbm_budget_bytes=1 << 20)
    setattr(cfg, field, value)
    with pytest.raises(T.ConfigError, match=re.escape(msg)):
        cfg.validate()


def test_no_cpu_fallback_without_device():
    if T.device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(T.CudaError):
        T.MultiStreamEngine(T.TierConfig(hbm_budget_bytes=1 << 20))


def test_gpu_limits_are_config_errors():
    with pytest.raises(T.ConfigError):
        T.MultiStreamEngine(T.TierConfig(hbm_budget_bytes=1 << 24, d_k=256, d_v=128))
    with pytest.raises(T.ConfigError):
        T.MultiStreamEngine(T.TierConfig(hbm_budget_bytes=1 << 24), ring_bytes=3)
    with pytest.raises(T.ConfigError):
        T.MultiStreamEngine(T.TierConfig(hbm_budget_bytes=1 << 20), heads_per_stream=9)
    with pytest.raises(T.ConfigError, match="record_stream"):
        T.MultiStreamEngine(T.TierConfig(hbm_budget_bytes=1 << 20), record_stream=3)


def test_null_handle_is_an_error():
    lib = L.lib()
    assert lib.ttkv_gpu_synchronize(None) == L.TTKV_EINVAL
    st = L.StateC()
    assert lib.ttkv_gpu_state(None, C.byref(st)) == L.TTKV_EINVAL
