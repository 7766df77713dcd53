"""B200-native FlashBlock attention hot path (arxiv 2602.05305).

Drop-in for the reference package's attention entry points
(flashblock.attention / flashblock.sparse / flashblock.policy), backed by
hand-written sm_100a CUDA kernels in libfb200.so behind a C ABI
(include/flashblock_b200.h).  No CPU fallback.
"""

from .attention import (AttnPartial, CacheEntry, DegenerateInputError, ExternalAttnCache,
                        ReusePreconditionError, attention_dense, attention_partial,
                        attention_streamed, attention_with_reuse, combine_partials,
                        merge_partials)
from .analysis import HeadGateCalibrator, pairwise_step_similarity
from .engine import FlashBlockAttention, KVCache, PagedKVCache
from .errors import BoundsError, ShapeError, StalenessError
from .policy import (MODES, CalibrationError, Decision, HeadGate, HeadGateTable, ReuseConfig,
                     count_updated_tokens, decide, refresh_schedule, unmask_schedule)
from .sparse import SparseMask, build_sparse_mask, sparse_attention_with_residual

__version__ = "0.1.0"

__all__ = [
    "AttnPartial", "CacheEntry", "DegenerateInputError", "ExternalAttnCache",
    "ReusePreconditionError", "attention_dense", "attention_partial", "attention_streamed",
    "attention_with_reuse", "combine_partials", "merge_partials", "FlashBlockAttention", "KVCache", "PagedKVCache",
    "BoundsError", "ShapeError", "StalenessError", "MODES", "Decision", "ReuseConfig",
    "count_updated_tokens", "decide", "refresh_schedule", "unmask_schedule", "SparseMask",
    "build_sparse_mask", "sparse_attention_with_residual", "CalibrationError", "HeadGate",
    "HeadGateTable", "HeadGateCalibrator", "pairwise_step_similarity",
]
