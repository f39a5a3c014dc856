"""B200-native (sm_100a) ReaLB MoE-layer hot path.

Host side (Python/PyTorch) mirrors the reference entry points of `moesim`
(policy.py: core + balancers; quant.py: fp4) and drives hand-written CUDA
kernels through the C-ABI library lib/librealb_b200.so (include/realb.h).
"""

from .policy import (  # noqa: F401
    STRATEGIES, ClusterConfig, ExpertPlacement, PlacementMismatchError, Precision, PrecisionPlan,
    RankLoad, RealbParams, aggregate_rank_loads, place_experts_static, plan_baseline, plan_for,
    plan_fp4_all, plan_realb, rank_loads_from_counts)
from .quant import QuantizationDomainError, quantize_blocks, quantize_nvfp4  # noqa: F401

__version__ = "0.1.0"
