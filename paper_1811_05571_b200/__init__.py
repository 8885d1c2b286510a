"""B200-native ADMM hot path of arXiv 1811.05571 (consensus / sectioning / hybrid lasso).

Drop-in for the reference admmsplit solver entry points; all arithmetic runs in the
sm_100a kernels of libadmm_b200.so.
"""
from .errors import (DeviceError, DimensionError, Error, FormatError, IndexError, IoError,  # noqa: F401
                     MetricsError, NumericalError, ParameterError, PartitionError, SingularityError,
                     NcclError, StateError)
from .cmat import cmat_info, read_cmat, read_cvec, write_cmat, write_cvec  # noqa: F401
from .comm import CommLedger, Convention, Method, per_node_elements, reduction_vs_consensus  # noqa: F401
from .solvers import (AdmmPlan, GramSolver, IterateSnapshot, PartitionSpec, ProblemKind,  # noqa: F401
                      RecoveryMetrics, ResidualTrace, SensingProblem, SolveOptions, SolveReport,
                      SolverConfig, adjoint_matvec, consensus_solve, hybrid_solve,
                      lasso_admm_reference, make_partition, matvec, recovery_metrics,
                      sectioning_solve, soft_threshold_vec)
from .generate import cra_matrix, cra_problem, cra_scenes, gen_problem  # noqa: F401

__all__ = [n for n in dir() if not n.startswith("_")]
