"""paper_2602_02108_b200 — B200-native OOMB hot path (arXiv 2602.02108).

Chunk-recurrent attention over a paged KV cache and a paged KV-gradient cache
(forward + recompute-backward), page scoring / top-k selection, behind the
reference's PagedCache / attention-operator API. Compute runs in liboomb.so
(sm_100a kernels, C ABI in include/oomb.h); there is no CPU fallback.
"""
from .config import ModelConfig, parse_model_config
from .errors import ConfigError, CudaError, IoError, OombError, ResidencyError, ShapeError, StateError

__all__ = [
    "ModelConfig", "parse_model_config", "ConfigError", "CudaError", "IoError", "OombError", "ResidencyError",
    "ShapeError", "StateError",
]


def __getattr__(name):
    # Operator modules import torch + liboomb lazily so config/errors stay light.
    if name in ("PagedCache", "SlotRange", "Gathered", "MemoryReport"):
        from . import paged_kv
        return getattr(paged_kv, name)
    if name in ("score_pages", "select_topk", "select_topk_row", "select_recent", "select_all", "attn_forward",
                "attn_backward", "AttnSaved", "AttnGrads", "Selection", "select_pages_topk", "select_topk_rows"):
        from . import attention
        return getattr(attention, name)
    raise AttributeError(name)
