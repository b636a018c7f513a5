"""B200-native (sm_100a) cosine-attention operator of Cotten4Rec (arXiv 2602.06935).

The hot path is libcotten.so (hand-written CUDA behind the C-ABI in
include/cotten.h); this package is its host-side mirror of the reference
operator API (attention.hpp:11-93).  Importing it loads the CUDA library and
fails loudly if it is missing — there is no CPU fallback.
"""
from ._lib import (CottenError, NumericError, ShapeError, UsageError,  # noqa: F401
                   load as _load)
from .ops import (AttentionCache, AttentionConfig, AttentionGrads, RowMask,  # noqa: F401
                  attention_backward, attention_forward, backward, cosine_attention_backward,
                  cosine_attention_fused, device_status, forward, fwd_bwd_host,
                  mechanism_from_string)

_load()

__all__ = [
    "AttentionCache", "AttentionConfig", "AttentionGrads", "RowMask", "UsageError", "ShapeError",
    "NumericError", "CottenError", "cosine_attention_fused", "cosine_attention_backward",
    "attention_forward", "attention_backward", "forward", "backward", "fwd_bwd_host",
    "device_status", "mechanism_from_string",
]
