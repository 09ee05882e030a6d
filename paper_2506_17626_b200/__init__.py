"""B200-native (sm_100a) drop-in for the featlsq hot path (arXiv 2506.17626):
assemble -> filter_system (truncated RRQR) -> precondition -> lsqr ->
recover_solution, with the same names, signatures and object surface as the
reference stage API (featlsq assembly.py:124, filtering.py:92/165/169,
solvers.py:87). Kernels: csrc/*.cu, C-ABI: include/featlsq_b200.h. The
package plugs into featlsq (`_featlsq.py`): value types, problem builders
and exceptions are featlsq's own; `integrate.enable()` rebinds featlsq's
stage functions to this package.
"""

from .assembly import (GlobalSystem, SolutionBlocks, SubdomainBlock, TestSet, apply,
                       apply_transpose, assemble, evaluate_solution, l1_error, make_test_set,
                       solution_matrix)
from .basis import ACTIVATIONS, FeatureBasis, init_basis
from .domains import Decomposition, Domain, decompose
from .errors import (CapExceededError, CoverageError, DegenerateSubdomainError, DeviceError,
                     DivergenceError, InvalidInputError, SingularFactorError)
from .filtering import (FilteredBlock, FilteredSystem, PreconditionedOperator, filter_system,
                        precondition, recover_solution)
from .linalg import PivotedQR, RandomSource, back_substitute, lattice_counts, qr_column_pivot
from .jets import Jet2, radial_jet
from .monitor import DeviceL1Error, test_error_fn
from ._featlsq import featlsq

# featlsq's own value types and problem builders (inputs of the stage API;
# the same objects, re-exported for convenience)
ConstraintRows = featlsq.ConstraintRows
LinearOperator2 = featlsq.LinearOperator2
ProblemSpec = featlsq.ProblemSpec
laplace_problem = featlsq.laplace_problem
oscillator_problem = featlsq.oscillator_problem
wave_problem = featlsq.wave_problem
from .solvers import (AdditiveSchwarz, ConvergenceMonitor, Operator, SolveResult, as_operator,
                      as_preconditioner, cg_normal, lsqr)

__version__ = "0.1.0"

__all__ = [
    "ACTIVATIONS", "CapExceededError", "ConstraintRows", "ConvergenceMonitor", "CoverageError",
    "Decomposition", "DegenerateSubdomainError", "DeviceError", "DivergenceError", "Domain",
    "FeatureBasis", "FilteredBlock", "FilteredSystem", "GlobalSystem", "InvalidInputError",
    "LinearOperator2", "Operator", "PivotedQR", "PreconditionedOperator", "ProblemSpec",
    "RandomSource", "SingularFactorError", "SolveResult", "SubdomainBlock", "apply",
    "apply_transpose", "as_operator", "assemble", "back_substitute", "decompose",
    "filter_system", "init_basis", "lattice_counts", "lsqr", "oscillator_problem",
    "precondition", "qr_column_pivot", "recover_solution",
    "DeviceL1Error", "Jet2", "SolutionBlocks", "TestSet", "evaluate_solution", "l1_error",
    "laplace_problem", "make_test_set", "radial_jet", "solution_matrix", "test_error_fn",
    "wave_problem", "AdditiveSchwarz", "as_preconditioner", "cg_normal",
]
