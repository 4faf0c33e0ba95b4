"""B200-native (sm_100a) log-domain Sinkhorn for point clouds.

Drop-in for the hot path of the reference package ``otkit`` (OTT paper,
arXiv 2201.12324): same public names for the linear entropic problem.
Every computation runs in libotk_sm100.so (hand-written CUDA for sm_100a,
C ABI in include/otk.h); there is no CPU fallback.
"""

from .barycenter import BarycenterOutput, BarycenterProblem, solve_barycenter
from .errors import DivergedError, OtkitError
from .geometry import (
    COST_FNS,
    DEFAULT_EPSILON_SCALE,
    DenseGeometry,
    EpsilonSchedule,
    Geometry,
    PointCloudGeometry,
)
from .sinkhorn import (
    BatchedSinkhornOutput,
    Coupling,
    LinearProblem,
    RegOTCost,
    SinkhornOutput,
    grad_points,
    grad_weights,
    reg_ot_cost,
    solve_sinkhorn,
    solve_sinkhorn_batched,
    transport_matrix,
)
from .sharded import ShardedProblem, reg_ot_cost_sharded, solve_sinkhorn_sharded

__version__ = "0.1.0"

__all__ = [
    "__version__",
    "OtkitError",
    "DivergedError",
    "Geometry",
    "DenseGeometry",
    "PointCloudGeometry",
    "EpsilonSchedule",
    "COST_FNS",
    "DEFAULT_EPSILON_SCALE",
    "LinearProblem",
    "SinkhornOutput",
    "Coupling",
    "RegOTCost",
    "solve_sinkhorn",
    "solve_sinkhorn_batched",
    "BatchedSinkhornOutput",
    "transport_matrix",
    "reg_ot_cost",
    "grad_weights",
    "grad_points",
    "solve_sinkhorn_sharded",
    "reg_ot_cost_sharded",
    "ShardedProblem",
    "BarycenterProblem",
    "BarycenterOutput",
    "solve_barycenter",
]
