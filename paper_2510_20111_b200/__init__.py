"""B200-native AsyncHZP hot path (arxiv 2510.20111).

Hierarchical ZeRO (Z1 optimizer / Z2 gradient / Z3 parameter sharding) with
layer-wise P2P-pull all-gather, fused reduce-scatter + Adam, and the
cyclic-slot async prefetch/consume scheduler mapped onto CUDA streams and
events; layer GEMMs on tcgen05.  Everything runs through libhzp_b200.so
(C-ABI: include/hzp_b200.h); importing this package fails loudly if the
library has not been built.
"""
from . import _native  # noqa: F401  (raises ImportError when the .so is missing)
from .hzp import (ASYNC, VANILLA, CostModel, ModelSpec, ParallelConfig, SchedError,  # noqa: F401
                  TaskGraph, ValidationError, build_process_groups, build_task_graph,
                  derive_prelaunch_depth, launch_plan, ledger, make_pools, memory_trace, shard_elems,
                  simulate, utilization_report, validate_config)
from .engine import BF16, FP32, GPT, MLP, EngineConfig, HzpEngine  # noqa: F401

__version__ = "0.1.0"
