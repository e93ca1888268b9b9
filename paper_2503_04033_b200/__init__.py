"""B200-native leaf-box reduction for the two-level HPS solver.

Drop-in for the leaf path of ``steklov`` (the reference package): same public
names for geometry, leaf templates, the build / load-reduction / solve stages
and the sparse backend; every per-leaf dense operation (operator assembly,
pivoted LU of A_ii, DtN Schur complement, interior solves) runs in the CUDA
engine ``libhps_leaf.so`` (sm_100a, FP64 DMMA tensor cores, TMA), with no CPU
fallback.
"""

from .condensation import (BatchSchedule, InterfaceSystem, SolveReport, build, estimate_workspace,
                           reduce_load, run_solve_stage, solve, solve_bvp)
from .errors import (ConfigError, CrossTermError, LeafSingularError, NativeUnavailableError,
                     NumericallySingularError, OracleCapExceededError, SolverError,
                     StructurallySingularError)
from .geometry import (DomainBox, Discretization, MeshConfig, ParameterMap, build_discretization,
                       leaf_neighbors, sinusoidal_map)
from .local_ops import (DROP_CORNERS, LEGENDRE_FACES, CoefficientField, LeafFactors, LeafTemplate,
                        build_leaf_factors, build_leaf_operator, cheb_diff_matrix, cheb_nodes,
                        face_interp_cheb_to_legendre, isotropic_field, laplace_field,
                        legendre_nodes)
from .problems import (ParabolicProblem, ProblemSpec, TimeStepConfig, crank_nicolson_run,
                       make_parabolic, make_problem, relative_l2_error)

__version__ = "0.1.0"
