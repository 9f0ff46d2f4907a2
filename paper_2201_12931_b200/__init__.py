"""B200-native drop-in for the MGPCG hot path of voxtop (arXiv 2201.12931).

Same public names as the reference package (pkg/src/voxtop/__init__.py:8-52);
the state-equation solve, its multigrid preconditioner and the per-iteration
design kernels run as hand-written sm_100a CUDA kernels in libvoxb200.so,
reached through the C ABI in include/voxb200.h.  There is no CPU fallback.
"""

from .errors import ConfigError, NumericalError, SetupError, SolverBreakdown, VolumeInfeasible
from .material import (
    ElementStiffness,
    MaterialModel,
    element_gravity_load,
    simp_scale,
    simp_scale_derivative,
    unit_stiffness,
)
from .mesh import (
    BoundarySpec,
    Box,
    GravitySpec,
    Region,
    RegionMask,
    StructuredGrid,
    build_grid,
    classify_regions,
    element_dofs_array,
    element_nodes,
    make_boundary,
)
from ._lib import lib as _native_lib  # noqa: F401  (fails loudly if the .so is missing)
from .device import DeviceGrid, DeviceVector
from .stiffness_op import OperatorState, apply, assemble_dense, diagonal, residual
from .hierarchy import MgHierarchy, build_hierarchy, max_feasible_levels
from .krylov import SolveReport, SolverConfig, jacobi_preconditioner, mgcg_solve, pcg
from .design import (
    DensityField,
    FilterWeights,
    OcResult,
    OptConfig,
    OptResult,
    Problem,
    RunRecord,
    build_filter,
    compliance,
    filter_sensitivities,
    initial_densities,
    oc_update,
    run,
    sensitivities,
    update_gravity_load,
)
from .multimaterial import (
    TwoMaterialRecord,
    TwoMaterialResult,
    initial_phases,
    run_two_material,
    sensitivities_two_material,
)

__version__ = "0.1.0"


def launch_count() -> int:
    """Kernels launched by libvoxb200 in this process."""
    return int(_native_lib.vt_launch_count())
