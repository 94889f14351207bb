"""paper_2009_12009_b200: B200-native MultiFab / FillBoundary / MLMG hot path.

A from-scratch rebuild of the data-parallel core of AMReX (arXiv 2009.12009)
as captured by the reference's Python package ``amrkit``: the public names
below mirror ``amrkit/__init__.py:11-45`` for the mesh path, plus the
``MultiFab`` alias and the ``MLMG`` geometric-multigrid Poisson solver.
Mesh data lives in PyTorch-owned CUDA memory; every operation on it is a
hand-written sm_100a kernel in libamrb.so (include/amrb.h).  There is no CPU
fallback.
"""

from . import counters
from .amr import AdvectionSolver, FaceFluxes, FluxRegister, fill_patch, snapshot_valid
from .boxes import Box, IndexType, IntVect, box_diff
from .comm import (
    Transport,
    TransportError,
    copy_into,
    device_reduce,
    fill_boundary,
    gather_global,
    parallel_copy,
    reduce,
    sum_boundary,
)
from .geometry import BoundaryRecord, Geometry, apply_domain_boundary
from .interlevel import average_down, coarsened_layout, interp_to_fine
from .layout import (
    BoxArray,
    BoxHash,
    DistributionMapping,
    default_costs,
    knapsack_distribute,
    load_stats,
    morton_key,
    sfc_distribute,
)
from .mlmg import MLMG, mg_hierarchy
from .multifab import ArrayView, Fab, FabArray, MultiFab
from .plotfile import (
    OutputMode,
    PlotfileHeader,
    WriteHandle,
    read_checkpoint,
    read_plotfile,
    write_checkpoint,
    write_plotfile,
)
from .plans import (
    CommPlan,
    CopyRecord,
    build_plan_copy,
    build_plan_copy_grown,
    build_plan_fill_boundary,
    build_plan_sum_boundary,
    plan_cache_clear,
)

__all__ = [
    "AdvectionSolver",
    "FaceFluxes",
    "FluxRegister",
    "fill_patch",
    "snapshot_valid",
    "OutputMode",
    "PlotfileHeader",
    "WriteHandle",
    "read_checkpoint",
    "read_plotfile",
    "write_checkpoint",
    "write_plotfile",
    "ArrayView",
    "BoundaryRecord",
    "Box",
    "BoxArray",
    "BoxHash",
    "CommPlan",
    "CopyRecord",
    "DistributionMapping",
    "Fab",
    "FabArray",
    "Geometry",
    "IndexType",
    "IntVect",
    "MLMG",
    "MultiFab",
    "Transport",
    "TransportError",
    "apply_domain_boundary",
    "average_down",
    "box_diff",
    "build_plan_copy",
    "build_plan_copy_grown",
    "build_plan_fill_boundary",
    "build_plan_sum_boundary",
    "coarsened_layout",
    "copy_into",
    "counters",
    "default_costs",
    "device_reduce",
    "fill_boundary",
    "gather_global",
    "interp_to_fine",
    "knapsack_distribute",
    "load_stats",
    "mg_hierarchy",
    "morton_key",
    "parallel_copy",
    "plan_cache_clear",
    "reduce",
    "sfc_distribute",
    "sum_boundary",
]

__version__ = "0.1.0"
