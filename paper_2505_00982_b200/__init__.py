"""B200-native DHO2 curvature-and-update hot path (arXiv 2505.00982).

libdho2gpu.so (hand-written sm_100a CUDA: tcgen05/TMA GEMMs on scaled-fp16 (hi, lo) operand pairs for
the HVP and gradient, fused Gram-Schmidt passes, fp64 tridiagonal eigensolve, fused FOSI/ADMM update,
NCCL collectives) behind a C ABI (include/dho2gpu.h); this package mirrors the
reference's C++ optimizer API (see api.py).
"""
from .api import *  # noqa: F401,F403
from .api import (AdmmState, ArgumentError, BaseConfig, BaseOptimizer, Batch, Context, Dataset, Deltas,
                  DimensionError, DistLanczosOptions, DivergenceError, EseResult, LanczosOptions, MlpOracle,
                  NumericError, QuadraticOracle, ShardedLanczosResult, Trainer, TrainerConfig, TrainingDiverged, admm_deltas,
                  admm_dual_update, admm_w_update, blobs_dataset, extract_ese_distributed, fosi_deltas,
                  lanczos_budget, lanczos_distributed, make_admm_state, quadratic_operator, shard_for_rank, train)
from ._lib import LIB_PATH, EXPORTED  # noqa: F401

__version__ = "0.1.0"
