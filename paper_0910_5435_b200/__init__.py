"""B200-native butterfly associated-Legendre engine (arXiv 0910.5435 hot path).

Host mirror of the reference's bfly:: interface over the C ABI in
include/bfly_b200.h; all transform arithmetic runs in the CUDA engine
(libbfly_b200.so).  Importing the package does not require a GPU; applying a
plan does, and fails loudly without one.
"""
from ._lib import (BflyCudaError, BflyError, BflyInvalidArgument, BflySerializationError,
                   LIB_PATH, SIGNATURES)
from .butterfly import (ButterflyPlan, PlanSet, PlanStats, apply, apply_transpose, build_glrow_plan,
                        build_glrow_planset, build_plan, chain_cols, forward, inverse, plan_stats)
from .sht import (SHT, coeff_index, coeff_offset, full_from_half, half_from_full, half_offset, pack_dense,
                  unpack_dense)
from .sharded import ShardedSHT, latitude_slabs, make_layout, partition_orders

__all__ = [
    "BflyCudaError", "BflyError", "BflyInvalidArgument", "BflySerializationError", "LIB_PATH",
    "SIGNATURES", "ButterflyPlan", "PlanSet", "PlanStats", "apply", "apply_transpose",
    "build_glrow_plan", "build_glrow_planset", "build_plan", "chain_cols", "forward", "inverse",
    "plan_stats", "SHT", "coeff_index", "coeff_offset", "pack_dense", "unpack_dense", "half_offset",
    "half_from_full", "full_from_half",
    "ShardedSHT", "latitude_slabs", "make_layout", "partition_orders",
]
