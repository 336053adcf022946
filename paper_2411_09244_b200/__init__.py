"""paper_2411_09244_b200 — B200-native (sm_100a) parareal hot path for the partially
explicit splitting scheme of arXiv 2411.09244 (reference package: paradiff).

Drop-in for the reference's online solver API; every solve runs in libpe
(hand-written FP64 DMMA / cluster kernels behind the C ABI in include/pe.h).
"""

from ._lib import LIB_PATH, NativeUnavailable, PeError  # noqa: F401
from .allatonce import (ImplicitAllAtOnce, TimeMatrixB, WaveformRelaxation,  # noqa: F401
                        WRResult, apply_S, apply_S_inverse, build_rhs, build_time_matrix,
                        wr_fine_solve)
from .engine import PeContext  # noqa: F401
from .msbasis import (CemSpace, CoarseSystem, build_cem_space, project_coarse,  # noqa: F401
                      project_load)
from .parareal import (AllAtOnceFine, ParerealConfig, ParerealEnsemble,  # noqa: F401
                       ParerealRun,
                       SequentialFine, build_fine_propagator, check_stop, initial_sweep,
                       max_state_diff, run_parareal, run_parareal_ensemble)
from .sharded import LibpeShardOps, run_parareal_sharded  # noqa: F401
from .stepping import (ConstantLoads, SplitPropagators, SplitState,  # noqa: F401
                       SplitTrajectory, TimeGrid, project_initial, split_energy)

__version__ = "0.1.0"
