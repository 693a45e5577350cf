"""B200-native Shift-Parallel transformer forward (arXiv 2507.11830).

Drop-in for the reference simulator's engine API (``shiftsim``,
/root/reference/pkg/src/shiftsim/__init__.py:73-137, hot-path subset): the
host side is Python/PyTorch, every arithmetic op is a hand-written sm_100a
kernel in ``libshiftpar.so`` behind the C-ABI of ``include/shiftpar.h``.
"""

from .config import ModelConfig, llama31_8b, llama33_70b, tiny_llama  # noqa: F401
from .engine import (  # noqa: F401
    Batch,
    BatchItem,
    BatchKind,
    CommEvent,
    Engine,
    ParallelMode,
    Sequence,
    ShiftPolicy,
    StepRecord,
    SwiftKvConfig,
    choose_mode,
    default_token_threshold,
    greedy_tokens,
    partition_heads,
)
from .errors import CacheOverflow, ConfigError, ContractViolation, LibraryMissing  # noqa: F401
from .fabric import DeviceGroup, LoopbackGroup, NcclGroup  # noqa: F401
from .flops import (FlopMeter, PassShape, flop_count, shard_bounds, shard_rows,  # noqa: F401
                    swiftkv_flop_ratio)
from .kv_cache import AXIS_ORDER, BlockAllocator, KvCache, KvPool, LayoutFingerprint  # noqa: F401
from .weights import (ModelWeights, TpShard, check_shard_containment, memory_report,  # noqa: F401
                      tp_shard_view)
from . import collectives, tensor_core  # noqa: F401,E402
from . import spec_decode  # noqa: F401,E402

__version__ = "0.1.0"
