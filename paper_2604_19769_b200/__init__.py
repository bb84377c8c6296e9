"""B200-native TTKV decode hot path (arxiv 2604.19769).

The product is libttkv_gpu.so (include/ttkv_gpu.h, sm_100a kernels under
csrc/); this package is its Python binding.  See DESIGN.md.
"""
from .engine import (ConfigError, CudaError, DecodeStepReport, Engine, Error, IntegrityError,
                     IoError, MultiStreamEngine, SelectionPolicy, SequencingError, ShapeError,
                     TierConfig, compressed_bytes_per_token, device_count, fast_capacity,
                     modeled_block_bytes, packed_bytes)

__all__ = ["ConfigError", "CudaError", "DecodeStepReport", "Engine", "Error", "IntegrityError",
           "IoError", "MultiStreamEngine", "SelectionPolicy", "SequencingError", "ShapeError",
           "TierConfig", "compressed_bytes_per_token", "device_count", "fast_capacity",
           "modeled_block_bytes", "packed_bytes"]
