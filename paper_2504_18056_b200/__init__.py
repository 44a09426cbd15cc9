"""B200-native hot path of gradient-guided 6-DoF Monte Carlo SLAM (arXiv 2504.18056).

The product is the C-ABI library ``libmcs.so`` (hand-written sm_100a CUDA, see
``include/mcs.h``); :mod:`paper_2504_18056_b200.mcs` is its thin ctypes binding.
"""
from .mcs import (ABI_VERSION, ALLOC_FN, CORR_CELL, CORR_NN27, FREE_FN, Allocator, Config, Context,
                  InprocTransport, MCSError, default_config,
                  header_symbols, load, nccl_unique_id, plan_ladder, plan_migration,
                  state_bytes_per_particle, TorchAllocator, TorchDistTransport, unpack_h21)

from .slam import MonteCarloSLAM, in_elevator

__all__ = ["MonteCarloSLAM", "in_elevator", "ABI_VERSION", "ALLOC_FN", "FREE_FN", "CORR_CELL",
           "CORR_NN27", "Allocator", "Config", "Context", "InprocTransport", "MCSError", "default_config",
           "header_symbols", "load", "nccl_unique_id", "plan_ladder", "plan_migration",
           "state_bytes_per_particle", "TorchAllocator", "TorchDistTransport", "unpack_h21"]
