"""B200-native GPUexplore hot path (arXiv 1801.05857): bucketed lock-free
state table with cooperative FINDORPUT, level-synchronous BFS with
on-device successor generation and deadlock detection, behind the Python
API of the reference package `ltsmc`.

Modules mirror the reference's (aut, network, statevec, hashtable,
explore, bench); the compute runs in libgx.so (csrc/, include/gx.h).
"""

__version__ = "0.1.0"

from .aut import Lts, NetworkDescription, ParseError, RuleSpec, parse_aut, parse_network  # noqa: F401
from .network import Network, NetworkError, SyncRule, build_network, load_network  # noqa: F401
from .hashtable import (  # noqa: F401
    EMPTY, CLAIMED, OCCUPIED_NEW, OCCUPIED_OLD, FOUND, INSERTED, TABLE_FULL, HALF_BUCKET, PLAIN,
    StateTable, TableConfig, TableFullError, slots_per_bucket,
)
from .explore import (  # noqa: F401
    COMPLETE, ITERATION_CAP, OUTCOME_TABLE_FULL, ExploreConfig, ExplorationReport, Explorer, explore,
)
