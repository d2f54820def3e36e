"""GGNN (arXiv 1912.01059) graph-based nearest-neighbour search, B200-native.

Drop-in for the reference package `graphann`
(/root/reference/pkg/src/graphann/__init__.py): same public names and
signatures; the hot path (query, hierarchical build, sharded search) runs as
hand-written sm_100a kernels in libggnn_b200.so behind a C ABI
(include/ggnn_b200.h).  There is no CPU fallback.
"""

from . import backend
from .config import BuildConfig, QueryConfig
from .data import (
    ConfigError,
    Dataset,
    FormatError,
    gen_synthetic,
    load_ids,
    load_vectors,
    squared_distance,
    write_ids,
    write_vectors,
)
from .graph import SENTINEL, AdjacencyLayer, GraphStats, Hierarchy
from .search import (
    BatchResult,
    QueryResult,
    batch_query,
    greedy_search,
    hierarchical_query,
    query,
    query_arrays,
    stopping_check,
    top_layer_seeds,
)
from .build import (
    BuildStats,
    build,
    build_base,
    compute_stats,
    merge_layer,
    partition_bottom,
    plan_geometry,
    refine_layer,
    select_points,
    symmetrize,
)

from .evaluate import GroundTruth, brute_force_oracle, consensus_at_k, k_recall_at, oracle_knn_graph, recall_at
from .index_file import IndexFormatError, load_index, save_index
from .shard import (
    ShardedIndex,
    batch_query_sharded,
    build_sharded,
    load_sharded,
    query_sharded,
    query_sharded_arrays,
    query_sharded_sequential,
    save_sharded,
)

__version__ = "0.1.0"
