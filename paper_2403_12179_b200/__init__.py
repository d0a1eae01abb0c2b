"""paper_2403_12179_b200 -- B200-native FillBoundary / ParallelCopy.

A drop-in for the ghost-cell exchange path of the reference package
``miniamr_core`` (AMReX/pyAMReX, arXiv 2403.12179): the same Python surface
(Box/IntVect/Geometry, BoxArray, DistributionMapping, MultiFab,
``fill_boundary`` / ``parallel_copy``, ``runtime_spawn``) over fab storage in
HBM, with a native plan builder and a single fused sm_100a copy kernel
behind the C ABI in include/ghostx.h (libghostx.so).
"""

from . import config
from ._native import GhostxError
from .comm import (Bus, CommPlan, CopySegment, PlanKey, RankContext, RankFailure, current_ctx,
                   current_rank, fill_boundary, global_reduce, parallel_copy, plan_build_fill_boundary,
                   runtime_spawn, MAX, MIN, SUM)
from .index_space import (CELL, NODE, Box, Geometry, IndexType, IntVect, box_diff, box_list_diff,
                          boxes_cover, coarsen, convert, empty_box, grow, intersect, num_pts,
                          periodic_shift_images, periodic_shifts, refine)
from .mesh import (BoxArray, DistributionMapping, Fab, FabView, MultiFab, decompose, fab_create,
                   fab_setval, multifab_define, storage_shape)

__version__ = "0.1.0"
from .bridge import BoundArray4, MfiAccessor, array_view, multifab_iter  # noqa: E402
from .comm import (build_gather_plan, gather_fabs, index_mapped_copy, prepare_fill_boundary,  # noqa: E402
                   prepare_parallel_copy)
from . import amr  # noqa: E402,F401
from .amr import LINEAR, PIECEWISE_CONSTANT, average_down, fill_patch, interp_box  # noqa: E402,F401
from . import heat  # noqa: E402,F401
from . import arena  # noqa: E402,F401
from . import kernels  # noqa: E402,F401
from .heat import advance_level, heat_step  # noqa: E402,F401
