"""B200-native H-matrix assembly + H-matvec (Helmholtz, elastodynamic U / T).

Drop-in for the reference ``hmatx`` hot path: the public names below keep the
reference signatures (``geometry.py`` / SPEC.md modules kernels, lowrank,
hmatrix, solve); the numerics run in ``libhmx.so`` (hand-written CUDA for
sm_100a + native C++ trees) through the C-ABI in ``include/hmx.h``.
"""

from .errors import (FallbackNeeded, PivotExhaustionError, SingularEvaluationError,  # noqa: F401
                     SnapshotCorruptError, SnapshotError, SnapshotVersionError, FactorizationError)
from .geometry import (AABB, AdmissibleLeaf, BlockTree, ClusterNode, ClusterTree, DenseLeaf,  # noqa: F401
                       PointCloud, Subdivided, build_block_tree, build_cluster_tree, diam_box,
                       dist_box, is_admissible, make_geometry, sparsity_pattern)
from .estimate import EstimatorReport, estimate  # noqa: F401
from .hierarchical_lu import LUFactors, formatted_addmul, hlu, lu_matvec, solve_direct, triangular_solve  # noqa: F401
from .hmatrix import HMatrix, StorageReport, assemble, block_errors, matvec, storage_report  # noqa: F401
from .kernels import (KernelSpec, Material, Wavenumbers, assemble_dense, elasto_t_block,  # noqa: F401
                      elasto_u_block, eval_elasto_t, eval_elasto_u, eval_scalar, scalar_block)
from .lowrank import (ACAConfig, ACAResult, BlockGenerator, LowRankFactor, aca_full, aca_partial,  # noqa: F401
                      aca_vector, numerical_rank, randomized_svd, recompress)
from .snapfile import snapshot  # noqa: F401
from .solve import GmresConfig, solve_gmres  # noqa: F401
