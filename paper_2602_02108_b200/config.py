"""ModelConfig — the fields of chunktrain::ModelConfig the hot path reads
(config.hpp:19-49), with the same invariants (ModelConfig::validate,
config.cpp:30-51) and the same key=value parser (config.cpp:86-133)."""
from __future__ import annotations

import dataclasses
from dataclasses import dataclass, field

from .errors import ConfigError

MODES = ("dense", "topk", "local")


@dataclass
class ModelConfig:
    n_layers: int = 2
    d_model: int = 64
    n_q_heads: int = 4
    n_kv_heads: int = 2
    head_dim: int = 16
    d_ff: int = 256
    vocab_size: int = 256
    chunk_size: int = 64     # C
    page_size: int = 16      # P
    attention_mode: list = field(default_factory=lambda: ["dense"])
    retrieval_budget: int = 128  # B tokens; B/P pages per query page in topk mode
    local_window: int = 4        # W pages
    rope_base: float = 10000.0
    seed: int = 0
    score_scale: bool = False

    def gqa_group(self) -> int:
        return self.n_q_heads // self.n_kv_heads

    def pages_per_chunk(self) -> int:
        return self.chunk_size // self.page_size

    def budget_pages(self) -> int:
        return self.retrieval_budget // self.page_size

    def mode_for_layer(self, layer: int) -> str:
        return self.attention_mode[0] if len(self.attention_mode) == 1 else self.attention_mode[layer]

    def validate(self) -> None:
        def req(ok, msg):
            if not ok:
                raise ConfigError("config: " + msg)

        req(self.n_layers >= 1, "n_layers must be >= 1")
        req(self.d_model >= 1, "d_model must be >= 1")
        req(self.n_q_heads >= 1 and self.n_kv_heads >= 1, "head counts must be >= 1")
        req(self.n_q_heads % self.n_kv_heads == 0, "n_q_heads must be divisible by n_kv_heads")
        req(self.head_dim >= 2 and self.head_dim % 2 == 0, "head_dim must be even (rotary pairs)")
        req(self.d_ff >= 1, "d_ff must be >= 1")
        req(self.vocab_size >= 2, "vocab_size must be >= 2")
        req(self.page_size >= 1, "page_size must be >= 1")
        req(self.chunk_size >= 1, "chunk_size must be >= 1")
        req(self.chunk_size % self.page_size == 0, "chunk_size must be divisible by page_size")
        req(self.retrieval_budget >= 0, "retrieval_budget must be >= 0")
        req(self.retrieval_budget % self.page_size == 0, "retrieval_budget must be divisible by page_size")
        req(self.local_window >= 0, "local_window must be >= 0")
        req(self.rope_base > 1.0, "rope_base must be > 1")
        req(len(self.attention_mode) in (1, self.n_layers), "attention_mode needs one entry or one per layer")
        for m in self.attention_mode:
            req(m in MODES, f"unknown attention mode '{m}' (expected dense|topk|local)")

    def replace(self, **kw) -> "ModelConfig":
        return dataclasses.replace(self, **kw)


_INT_KEYS = ("n_layers", "d_model", "n_q_heads", "n_kv_heads", "head_dim", "d_ff", "vocab_size", "chunk_size",
             "page_size", "retrieval_budget", "local_window", "seed")


def parse_model_config(text: str) -> ModelConfig:
    """`key = value` lines, '#' comments, unknown keys are errors (config.cpp:86-133)."""
    cfg = ModelConfig()
    for lineno, line in enumerate(text.splitlines(), 1):
        line = line.split("#", 1)[0].strip()
        if not line:
            continue
        if "=" not in line:
            raise ConfigError(f"config line {lineno}: expected key = value")
        key, val = (s.strip() for s in line.split("=", 1))
        if key in _INT_KEYS:
            try:
                setattr(cfg, key, int(val))
            except ValueError:
                raise ConfigError(f"config: key '{key}' expects an integer, got '{val}'") from None
        elif key == "rope_base":
            try:
                cfg.rope_base = float(val)
            except ValueError:
                raise ConfigError(f"config: key '{key}' expects a number, got '{val}'") from None
        elif key == "score_scale":
            cfg.score_scale = int(val) != 0
        elif key == "attention_mode":
            modes = []
            for item in val.split(","):
                item = item.strip()
                item = "topk" if item == "topk_sparse" else item
                if item not in MODES:
                    raise ConfigError(f"unknown attention mode '{item}' (expected dense|topk|local)")
                modes.append(item)
            if not modes:
                raise ConfigError("config: attention_mode list is empty")
            cfg.attention_mode = modes
        else:
            raise ConfigError(f"config: unknown key '{key}'")
    cfg.validate()
    return cfg
