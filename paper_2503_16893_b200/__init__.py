"""B200-native (sm_100a) SamuLLM sampling-then-simulation estimator (arXiv 2503.16893).

The computation lives in libsamu.so (CUDA C++, C ABI in include/samu.h); `binding` is the thin
ctypes layer over it.
"""
from .binding import (LocalGroup, Samu, SamuError, lib, recs_to_numpy, rec_flops, samu_nccl_unique_id,  # noqa: F401
                      samu_shard_classes, samu_shard_plan)
