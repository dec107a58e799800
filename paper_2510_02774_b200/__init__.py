"""B200-native GRNND (arXiv 2510.02774) graph construction -- the drop-in for
the reference package's build path (``grnnd.build`` and its stepwise API).

Hand-written sm_100a CUDA (libgrnnd_b200.so, C ABI in include/grnnd_b200.h)
does all the work; PyTorch supplies device memory and streams.  Importing
this package fails loudly when the library is not built.
"""

from .core import (
    TOMBSTONE,
    BuildParams,
    Dataset,
    DoubleBufferPool,
    Graph,
    NeighborEntry,
    generate,
    validate_params,
)
from .errors import (
    DeviceError,
    DimensionMismatch,
    EmptyGraph,
    FormatError,
    GrnndError,
    LengthMismatch,
    ParamError,
    SelfInsert,
)

__version__ = "0.1.0"


from .builder import (  # noqa: E402  (loads libgrnnd_b200.so; raises if it is not built)
    BuildState,
    RoundStats,
    build,
    build_fixed_degree,
    cooperative_insert,
    effective_params,
    finalize_graph,
    init_neighbors,
    reverse_edge_sampling,
    rng_redirect_check,
    update_round,
    validate_state,
)
from .sequential import CandidateList, build_seq, update_neighbors_seq  # noqa: E402
from .search import (  # noqa: E402
    SearchParams,
    brute_force_knn,
    brute_force_knn_batch,
    greedy_search,
    mean_recall,
    recall_at_k,
    search_batch,
)

__all__ = [
    "BuildParams", "BuildState", "Dataset", "DeviceError", "DimensionMismatch", "DoubleBufferPool",
    "EmptyGraph", "FormatError", "Graph", "GrnndError", "LengthMismatch", "NeighborEntry", "ParamError",
    "RoundStats", "SelfInsert", "TOMBSTONE", "build", "build_fixed_degree", "cooperative_insert",
    "effective_params", "finalize_graph", "generate", "init_neighbors", "reverse_edge_sampling",
    "rng_redirect_check", "update_round", "validate_params", "validate_state",
    "SearchParams", "brute_force_knn", "brute_force_knn_batch", "greedy_search", "mean_recall", "recall_at_k",
    "search_batch", "CandidateList", "build_seq", "update_neighbors_seq",
]
