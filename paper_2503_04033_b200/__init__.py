"""B200-native leaf-box reduction for the two-level HPS solver (drop-in for steklov's leaf path)."""

from .errors import (ConfigError, CrossTermError, LeafSingularError, NativeUnavailableError,
                     NumericallySingularError, SolverError, StructurallySingularError)
from .local_ops import (DROP_CORNERS, LEGENDRE_FACES, CoefficientField, LeafFactors, LeafTemplate,
                        build_leaf_factors, build_leaf_operator, cheb_diff_matrix, cheb_nodes,
                        face_interp_cheb_to_legendre, isotropic_field, laplace_field, legendre_nodes)

__version__ = "0.1.0"
