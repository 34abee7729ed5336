"""B200-native two-level spectral Schwarz PCG for high-contrast elasticity.

Drop-in for the solve path of the reference package ``mselast`` (EH, EH+Rot,
EH+Rot;Rand, HH, HH+Rot variants) and its SIMP caller: the public names below
mirror ``mselast.grid``, ``mselast.assembly``, ``mselast.schwarz``,
``mselast.krylov`` and ``mselast.topopt``; every
solver call runs in hand-written sm_100a kernels behind the C ABI
``include/msgpu.h`` (``libmsgpu.so``).  There is no CPU fallback.
"""

from .grid import FineMesh, CoarsePartition, Patch, build_fine_mesh, build_coarse_partition
from .assembly import (CoefficientField, LoadSpec, ElasticityOperator, assemble_elasticity,
                       build_load_vector, element_stiffness_elasticity, simp_modulus,
                       vector_dirichlet_dofs)
from .schwarz import (VARIANTS, GPU_VARIANTS, EigOptions, IdentityPreconditioner,
                      TwoLevelPreconditioner, build_preconditioner, get_variant)
from .krylov import SolveReport, estimate_condition, pcg_solve
from .solve import solve_spec
from . import topopt
from .topopt import (DensityFilter, OptimizeConfig, OptimizationResult, ReusePolicy,
                     compliance_and_sensitivity, oc_update, optimize)



def release_cached_memory():
    """Return the device memory kept by the library's block cache to the driver
    (e.g. before large allocations outside this package); returns the bytes freed."""
    from ._lib import cache_trim

    held = cache_trim(False)
    cache_trim(True)
    return held


__all__ = [n for n in dir() if not n.startswith("_")]
