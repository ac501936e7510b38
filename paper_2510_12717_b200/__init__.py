"""paper_2510_12717_b200 — B200-native batched RTI-MPC solver (Residual MPC hot path).

Host-side mirror of the reference's batch runtime interface (rmpc::BatchRunner,
/root/reference/proj/include/rmpc/batch.hpp:24-46) over the C ABI in include/rmpc_b200.h.
The compute runs only in the sm_100a kernel of lib/librmpc_b200.so; there is no CPU fallback:
importing works without a GPU, but constructing a BatchRunner fails loudly if the library or
a CUDA device is missing.
"""
from __future__ import annotations

from .abi import (NC, NF, NJ, NQ, NV, SOLUTION_DTYPE, STAGE_NAMES, STATUS_DIVERGED,  # noqa: F401
                  STATUS_NONFINITE_INPUT, STATUS_OK, STATUS_SINGULAR, Model, Settings, Timing,
                  default_model, default_settings, gait_row, standing_gait_row)
from .runtime import SOA_FIELDS, BatchRunner, RmpcError, from_soa, library, load_library, to_soa  # noqa: F401
from .synthetic import synthetic_batch  # noqa: F401
from .env import Env, EnvConfig, Policy, default_env_config  # noqa: F401

__all__ = ["BatchRunner", "RmpcError", "Model", "Settings", "Timing", "default_model",
           "default_settings", "gait_row", "standing_gait_row", "synthetic_batch",
           "SOLUTION_DTYPE", "load_library", "library", "Env", "EnvConfig", "Policy", "default_env_config",
           "to_soa", "from_soa", "SOA_FIELDS"]
