"""B200-native randomized t-SVT and nonconvex tensor-recovery hot path.

Drop-in for the hot path of the reference package ``tenrec``
(/root/reference/pkg/src/tenrec): the same public names and call signatures
for the randomized low-rank tensor approximation and the ADMM solvers, backed
by hand-written sm_100a CUDA kernels behind the C ABI in
``include/tenrec_b200.h``.  There is no CPU fallback.
"""

from .penalties import (PENALTY_NAMES, L1, MCP, SCAD, CappedLq, Firm, LogPenalty, Lq, Penalty,
                        make_penalty)
from .gradient import GradientSet, solve_grad_system
from .onebit import (ObservationSet, data_fit_update, gnobhtc, gnobrhtc, naive_estimate,
                     onebit_observe)
from .shard import (DeviceAllreduce, DeviceComm, gnhtc_sharded, gnhtsvt_randomized_sharded,
                    gnrhtc_sharded, shard_range)
from .sketch import (BLBPDiagnostics, SketchConfig, TuckerFactors, ad_rsthosvd_blbp,
                     gnhtsvt_randomized, rsthosvd_bki)
from .solvers import SolveReport, SolverConfig, default_lambda, gnhtc, gnrhtc
from .transform import DEFAULT_TRANSFORM, Transform, TransformError

__version__ = "0.1.0"

__all__ = [
    "PENALTY_NAMES", "L1", "MCP", "SCAD", "CappedLq", "Firm", "LogPenalty", "Lq", "Penalty",
    "make_penalty", "SketchConfig", "TuckerFactors", "BLBPDiagnostics", "gnhtsvt_randomized",
    "rsthosvd_bki", "ad_rsthosvd_blbp",
    "DEFAULT_TRANSFORM", "Transform", "TransformError", "SolveReport", "SolverConfig",
    "default_lambda", "gnhtc", "gnrhtc", "ObservationSet", "data_fit_update", "gnobhtc",
    "gnobrhtc", "naive_estimate", "onebit_observe", "GradientSet", "solve_grad_system", "DeviceAllreduce", "gnhtsvt_randomized_sharded", "shard_range",
    "DeviceComm", "gnrhtc_sharded", "gnhtc_sharded",
]
