"""B200-native engine for the INLA hyperparameter objective f(theta) and the
Takahashi selected inversion (arxiv 2204.04678 hot path).

Drop-in surface of the reference package ``parinla`` for the hot path:
``ObjectiveEvaluator``, ``fd_gradient``, ``parallel_line_search``,
``selected_inverse`` / ``latent_marginals`` keep their signatures; the
arithmetic runs in the in-tree CUDA library ``libpinla.so`` (sm_100a).
"""

from .errors import (
    BatchError,
    BudgetError,
    ConfigError,
    DimensionMismatch,
    EngineError,
    EvaluationError,
    InnerDivergence,
    LineSearchFailure,
    NotPositiveDefinite,
    ParinlaError,
    RobustFitError,
    StructureError,
)
from .model import (
    Component,
    HyperParams,
    LatticeGraph,
    ModelSpec,
    assemble_prior_precision,
    build_design,
    likelihood_terms,
    log_prior_hyper,
)
from .objective import GaussianApprox, ObjectiveEvaluator, ObjectiveValue
from .runtime import (
    SERIAL,
    ThreadBudget,
    default_budget,
    parse_budget,
    reset_runtime_stats,
    run_batch,
    runtime_stats,
)
from .sparse import SparseSymMatrix

__version__ = "0.1.0"
