"""B200-native SPED hot path (arXiv 2207.14589).

Drop-in for the reference ``specgap`` package's hot path: graph ->
Laplacian CSR -> dilation-polynomial apply -> mu-EigenGame / Oja step ->
embedding + k-means, with every hot op a hand-written sm_100a CUDA kernel in
``libsped.so`` (C ABI: ``include/sped.h``).  There is no CPU fallback.
"""

from .graph import (
    Graph,
    LaplacianOperator,
    DegreeBounds,
    build_laplacian,
    laplacian_matvec,
    dense_laplacian,
    degree_bounds,
)
from .walks import (
    SamplerConfig,
    estimate_power_matvec,
    estimate_polynomial_matvec,
    WalkOracle,
)
from .transforms import (
    SpectralTransform,
    TransformedOperator,
    scalar_map,
    polynomial_coefficients,
    choose_lambda_star,
    exact_transform_dense,
    apply_transform_matvec,
    make_reversed_operator,
    term_schedule,
    TRANSFORM_KINDS,
)
from .solvers import (
    EigenState,
    SolverConfig,
    MetricRow,
    SolverRun,
    StepWorkspace,
    init_state,
    orthonormalize,
    oja_step,
    mu_eg_step,
    make_stochastic_oracle,
    run_solver,
    run_to_csv,
)
from .metrics import (
    GroundTruth,
    dense_eig,
    graph_ground_truth,
    subspace_error,
    eigenvector_streak,
    eigengaps,
    kmeans_cluster,
    cluster_accuracy,
    match_labels,
    principal_angles,
    ritz_values,
)
from .sampling import EdgeBatchOracle, pcg64_draw, host_draw
from . import generators

__version__ = "0.1.0"
