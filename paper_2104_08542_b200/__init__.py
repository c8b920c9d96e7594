"""B200-native ScaleFreeCTR embedding hot path (arXiv 2104.08542).

The product is ``libsfctr_b200.so`` (sm_100a kernels + C-ABI, see
include/sfctr_b200.h); ``sfctr`` is its Python ctypes binding.
"""
from . import sfctr  # noqa: F401
from .sfctr import (  # noqa: F401
    BatchSource, CacheBuffer, Config, ConfigError, CudaError, DataError, LogicError, NcclError, RunError, SfctrError,
    CriteoReader, SyntheticGenerator, Trainer, VirtualSparseId, allreduce_bytes, derive_seed, device_count,
    fnv1a64, initial_embedding, model_forward_backward, nccl_unique_id, virtual_sparse_id)
