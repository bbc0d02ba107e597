"""B200-native IceCache decode hot path (arXiv 2604.10539).

Drop-in for the reference package's cache/index API on the decode path:
DCI-tree build and insert, query-aware top-k page selection, page union and
sparse paged attention run as sm_100a kernels behind a C ABI
(include/icecache_b200.h); this package is the Python host side.
"""

from .errors import (ConfigError, ConsistencyError, DegenerateQueryError, IceCacheError, InputError,
                     InvariantViolation, PolicyError, ScaleViolationError)
from .forest import DeviceForest, ForestCaps, dense_attention, entropy_words
from .attention import AttentionOutput, HeadGroup, full_attention, gqa_union, sparse_attention
from .dci import (PARENT_BUDGET, SENTINEL_LEVEL, DciTree, KeyScale, SearchBudget, assign_level, dci_indexing,
                  query_raw, transform_query)
from .engine import Engine, EngineConfig, StepMetrics, prefill
from .pagestore import Page, PageTable, TierStore, TransferStats, TreePageTable, find_page_index
from .workload import DecodeStep, Workload, WorkloadSpec, generate_workload

__version__ = "0.1.0"
