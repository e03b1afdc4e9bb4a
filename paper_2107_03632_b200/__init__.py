"""B200-native explicit RBF-FD Poisson time loop (arXiv 2107.03632).

Drop-in for the solve path of the reference package ``rbffd``
(pkg/src/rbffd/__init__.py:8-48 re-exports; solver.py:168-311): same names,
argument meaning and exceptions, with the time loop running in the sm_100a
CUDA library behind the C ABI of include/rbffd_b200.h.
"""

from .errors import DegenerateStencilError, DeviceError, InstabilityError, ParameterError, SteadyStateTimeout
from .problem import (
    NodeSet,
    ShapeStore,
    StencilSet,
    closed_form_solution,
    forcing,
    load_fixture,
    load_problem,
    save_problem,
    node_count_for_spacing,
    spacing_for_node_count,
)
from .solver import (
    Plan,
    SolveConfig,
    SolveReport,
    apply_dirichlet,
    clear_plan_cache,
    error_norms,
    explicit_step,
    prepare_problem,
    run_time_loop,
    save_report_json,
    save_solution_csv,
    stability_bound,
)

__version__ = "0.1.0"
