"""FlashOmni hot path, B200-native (sm_100a tcgen05/TMEM/TMA kernels).

Drop-in for the operator API of the reference `omniattn` package
(pkg/src/omniattn/__init__.py): sparse-symbol codec, sparse_attention,
GEMM-Q (project_q), GEMM-O (project_out_update / project_out_dispatch) and the
feature cache — batched over heads and resident in HBM. The compute runs in
the C-ABI library `_fo_b200.so` (include/flashomni_b200.h); there is no CPU
fallback.
"""

from .errors import (
    BoundsError,
    ConsistencyError,
    DeviceError,
    EngineError,
    ParameterError,
    ShapeError,
    StateError,
)
from .symbols import (
    SYMBOL_FORMAT_VERSION,
    DeviceSymbols,
    SymbolBuffer,
    build_symbols,
    ceil_div,
    decode_reduction,
    decode_run,
    decode_spatial,
    encode_cache_mask,
    encode_skip_mask,
    encode_symbols,
)
from .attention import (
    AttnCounters,
    CacheEntry,
    FeatureCache,
    OnlineSoftmaxState,
    dense_attention_update,
    forecast,
    forecast_coefficients,
    online_softmax_finalize,
    online_softmax_update,
    sparse_attention,
    update_entry,
)
from .gemm import (
    CachedBias,
    GemmCounters,
    pack_w_out,
    pack_w_q,
    pack_w_qkv,
    project_out_dispatch,
    project_out_update,
    project_q,
    project_qkv,
    rope_tables,
)
from .gemm_ref import ReferenceCachedBias
from .pipeline import (
    HostStepper,
    LayerParams,
    LayerState,
    dispatch_step,
    new_layer_state,
    project_kv,
    shard_heads,
    update_step,
)
from .costs import (
    CostReport,
    StepCost,
    account_run,
    sparsity,
    theoretical_speedup_attention,
    theoretical_speedup_gemm_o,
)
from .engine import (
    Engine,
    EngineConfig,
    RunResult,
    SyntheticWorkload,
    config_from_dict,
    dense_reference,
    max_rel_error,
    run,
    synthetic_workload,
)
from .policy import (
    CompressedAttnMap,
    MaskPolicy,
    compressed_attention,
    degrade_to_full_cache,
    generate_masks,
    generate_masks_heads,
    ramp_threshold,
    select_cached_blocks,
    select_skip_blocks,
    text_to_vision_guidance,
    vision_to_text_contribution,
)
from .tensor import dense_attention, matmul, mean_pool_blocks, rms_norm, rope, row_softmax
from ._kernels import available_backends, get_backend

__version__ = "0.1.0"


def backend_name():
    return "b200"


__all__ = [n for n in dir() if not n.startswith("_")]
