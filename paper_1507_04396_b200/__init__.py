"""B200-native pMMF stage loop (arXiv 1507.04396): hand-written sm_100a
kernels behind the reference's factorize / MmfOperator / solver interface."""
from .api import (  # noqa: F401
    BlockedSparseMatrix,
    ClusterParams,
    FactorizeParams,
    MmfFactorization,
    MmfOperator,
    Partition,
    factorize,
    kernel_launches,
    library,
    result_handle_from,
    workload_aniso_grid,
    workload_dense_spd,
    workload_rbf,
    workload_rmat,
)
