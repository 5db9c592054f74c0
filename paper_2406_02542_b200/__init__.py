"""B200-native Loki decode-time sparse attention (arXiv 2406.02542).

Drop-in for the hot path of the reference package ``lokiattn``: the public
names below match ``lokiattn/__init__.py:13-65`` for PCA calibration and
transform, Loki attention with k_f / d_f, and the pre/post-rotary
compositions.  The arithmetic runs in hand-written sm_100a CUDA
(libloki_b200.so, C ABI in include/loki_b200.h); there is no CPU fallback.
"""

__version__ = "0.1.0"

from .attention import (
    DecodeGraph,
    KvCache,
    LokiConfig,
    LokiDecoder,
    LokiDiagnostics,
    RotaryComposition,
    cache_append,
    dense_decode,
    exact_topk_attention,
    loki_attention,
    loki_decode,
    loki_rank_and_attend,
    pca_attn,
    resolve_fraction,
    transform_step,
    vanilla_attention,
)
from .calibration import (
    ProjectionSet,
    build_projection,
    compute_covariance,
    eigh_symmetric,
    rank_at_v,
    stack_projections,
)
from .dataio import (
    KeyDumpHeader,
    SyntheticSpec,
    gen_synthetic_keys,
    read_key_dump,
    read_projection,
    write_key_dump,
    write_projection,
)
from .errors import (
    BudgetError,
    DataError,
    DomainError,
    LokiCudaError,
    LokiError,
    ShapeError,
    UnsupportedShapeError,
    UsageError,
)
from .kernels import (
    TileSpec,
    dense_weighted_sum_kernel,
    gather_copy_scores_reference,
    gathered_score_kernel,
    gathered_weighted_sum_kernel,
    sliced_score_kernel,
)
from .linalg import canonicalize_indices, softmax_row, softmax_rows, topk_indices, topk_rows
from .metrics import (
    AgreementCell,
    AgreementStats,
    agreement_sweep,
    exact_speedup,
    jaccard_topk,
    score_error,
    theoretical_speedup,
)
from .rope import RopeParams, rope_angles, rope_apply, rope_apply_rows

__all__ = [name for name in dir() if not name.startswith("_")]
