"""Model configuration and presets.

``ModelConfig`` keeps the reference's fields (model.py:41-60: n_layers,
n_heads, head_dim, ffn_dim, vocab_size, max_seq) and adds the Llama features
the north star needs: ``n_kv_heads`` (GQA), ``pos`` ("rope" | "sinusoidal"),
``mlp`` ("swiglu" | "gelu"), ``norm_eps`` and the RoPE parameters.  The
reference's own model family is ``pos="sinusoidal", mlp="gelu",
n_kv_heads=None, norm_eps=1e-6``.
"""

from __future__ import annotations

from dataclasses import dataclass, replace
from typing import Optional

from .errors import ConfigError

LLAMA3_ROPE_SCALING = {
    "factor": 8.0,
    "low_freq_factor": 1.0,
    "high_freq_factor": 4.0,
    "original_max_position_embeddings": 8192,
}


@dataclass(frozen=True)
class ModelConfig:
    n_layers: int = 4
    n_heads: int = 8
    head_dim: int = 16
    ffn_dim: int = 512
    vocab_size: int = 256
    max_seq: int = 4096
    n_kv_heads: Optional[int] = None
    pos: str = "sinusoidal"
    mlp: str = "gelu"
    norm_eps: float = 1e-6
    rope_theta: float = 500000.0
    rope_scaling: Optional[dict] = None
    name: str = "custom"

    @property
    def hidden(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_heads(self) -> int:
        return self.n_heads if self.n_kv_heads is None else self.n_kv_heads

    @property
    def group(self) -> int:
        return self.n_heads // self.kv_heads

    def validate(self) -> "ModelConfig":
        for k in ("n_layers", "n_heads", "head_dim", "ffn_dim", "vocab_size", "max_seq"):
            if getattr(self, k) < 1:
                raise ConfigError(f"model.{k} must be >= 1")
        if self.n_heads % self.kv_heads:
            raise ConfigError("n_heads must be a multiple of n_kv_heads")
        if self.pos not in ("rope", "sinusoidal") or self.mlp not in ("swiglu", "gelu"):
            raise ConfigError("pos must be rope|sinusoidal and mlp swiglu|gelu")
        if self.head_dim not in (32, 64, 128):
            raise ConfigError("head_dim must be 32, 64 or 128 (attention kernels)")
        if self.hidden % 8 or self.ffn_dim % 8:
            raise ConfigError("hidden and ffn_dim must be multiples of 8")
        return self

    def check_world(self, world_size: int) -> None:
        """Divisibility the head/ffn/vocab partition needs (config.py:48-75)."""
        for name, dim in (("n_heads", self.n_heads), ("n_kv_heads", self.kv_heads),
                          ("ffn_dim", self.ffn_dim), ("vocab_size", self.vocab_size)):
            if dim % world_size:
                raise ConfigError(f"{name}={dim} must be divisible by world_size={world_size}")
        if self.mlp == "swiglu" and (self.ffn_dim // world_size) % 128:
            raise ConfigError("SwiGLU needs ffn_dim / world_size to be a multiple of 128")

    def with_(self, **kw) -> "ModelConfig":
        return replace(self, **kw)


def tiny_llama(**kw) -> ModelConfig:
    """BASELINE configs[0] (C1): 4 layers, hidden 256, 8 q / 2 kv heads, f 1024."""
    base = dict(n_layers=4, n_heads=8, n_kv_heads=2, head_dim=32, ffn_dim=1024, vocab_size=256,
                max_seq=4096, pos="rope", mlp="swiglu", norm_eps=1e-5, rope_theta=500000.0,
                rope_scaling=LLAMA3_ROPE_SCALING, name="tiny-llama")
    base.update(kw)
    return ModelConfig(**base).validate()


def llama31_8b(**kw) -> ModelConfig:
    """Llama-3.1-8B geometry (BASELINE configs[1], [2], [4])."""
    base = dict(n_layers=32, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336,
                vocab_size=128256, max_seq=32768, pos="rope", mlp="swiglu", norm_eps=1e-5,
                rope_theta=500000.0, rope_scaling=LLAMA3_ROPE_SCALING, name="llama-3.1-8b")
    base.update(kw)
    return ModelConfig(**base).validate()


def llama33_70b(**kw) -> ModelConfig:
    """Llama-3.3-70B geometry (BASELINE configs[3])."""
    base = dict(n_layers=80, n_heads=64, n_kv_heads=8, head_dim=128, ffn_dim=28672,
                vocab_size=128256, max_seq=8192, pos="rope", mlp="swiglu", norm_eps=1e-5,
                rope_theta=500000.0, rope_scaling=LLAMA3_ROPE_SCALING, name="llama-3.3-70b")
    base.update(kw)
    return ModelConfig(**base).validate()
