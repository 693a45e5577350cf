"""Oracle model: config, seeded weights, head partition, dense forward.

Restates ``/root/reference/pkg/src/shiftsim/model.py``:

* ``compat_config`` / ``init_weights_compat`` — ModelConfig (:41-60) and the
  single-stream draw order of ``init_weights`` (:89-112), bit-identical;
* ``partition_heads`` — :186-193;
* ``forward_reference`` — :310-354 (embed + positions, pre-norm blocks,
  final norm, head), bit-identical in compat mode;
* ``greedy_token`` — :303-307 (argmax, lowest index wins ties).

Llama mode extends the same structure with ``n_kv_heads`` (GQA), RoPE and
SwiGLU, per-tensor seeded streams (so 8B/70B tensors can be drawn
independently) and bf16-rounded weights (the exact values the
GPU holds).  Weights use the reference's ``x @ W`` orientation: W is [in, out].
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Dict, List, Optional, Sequence, Tuple

import numpy as np

from .kvcache import OracleKvCache
from .prims import (
    OracleContractError,
    attend_cached,
    bf16_round,
    gelu,
    matmul,
    rms_norm,
    rope_apply,
    rope_tables,
    silu,
    sinusoidal_positions,
)

WEIGHT_SCALE = 0.02  # model.py:86

LLAMA3_SCALING = {
    "factor": 8.0,
    "low_freq_factor": 1.0,
    "high_freq_factor": 4.0,
    "original_max_position_embeddings": 8192,
}


@dataclass(frozen=True)
class OracleConfig:
    n_layers: int = 4
    n_heads: int = 8
    head_dim: int = 16
    ffn_dim: int = 512
    vocab_size: int = 256
    max_seq: int = 4096
    n_kv_heads: Optional[int] = None      # None -> MHA (reference)
    pos: str = "sinusoidal"               # "sinusoidal" (reference) | "rope"
    mlp: str = "gelu"                     # "gelu" (reference) | "swiglu"
    norm_eps: float = 1e-6                # tensor_core.py:115 default
    rope_theta: float = 500000.0
    rope_scaling: Optional[dict] = None

    @property
    def hidden(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def kv_heads(self) -> int:
        return self.n_heads if self.n_kv_heads is None else self.n_kv_heads

    @property
    def group(self) -> int:
        return self.n_heads // self.kv_heads

    @property
    def compat(self) -> bool:
        return self.pos == "sinusoidal" and self.mlp == "gelu" and self.kv_heads == self.n_heads

    def validate(self) -> "OracleConfig":
        for k in ("n_layers", "n_heads", "head_dim", "ffn_dim", "vocab_size", "max_seq"):
            if getattr(self, k) < 1:
                raise OracleContractError(f"{k} must be >= 1")
        if self.n_heads % self.kv_heads:
            raise OracleContractError("n_heads must be a multiple of n_kv_heads")
        if self.pos not in ("sinusoidal", "rope") or self.mlp not in ("gelu", "swiglu"):
            raise OracleContractError("unknown pos/mlp kind")
        if self.hidden % 2 or self.head_dim % 2:
            raise OracleContractError("hidden and head_dim must be even")
        return self


def compat_config(**kw) -> OracleConfig:
    """The reference's own model family (MHA / sinusoidal / GeLU / eps 1e-6)."""
    return OracleConfig(**kw).validate()


def llama_tiny_config(**kw) -> OracleConfig:
    """C1 'tiny Llama' (BASELINE.json configs[0]): L4, h256, 8q/2kv heads, f1024."""
    base = dict(n_layers=4, n_heads=8, n_kv_heads=2, head_dim=32, ffn_dim=1024,
                vocab_size=256, max_seq=4096, pos="rope", mlp="swiglu",
                norm_eps=1e-5, rope_theta=500000.0, rope_scaling=LLAMA3_SCALING)
    base.update(kw)
    return OracleConfig(**base).validate()


@dataclass
class OracleWeights:
    config: OracleConfig
    dtype: np.dtype
    seed: int
    embed: np.ndarray                 # [V, h]
    layers: List[Dict[str, np.ndarray]]
    final_gain: np.ndarray            # [h]
    head: np.ndarray                  # [h, V]
    rope: Optional[np.ndarray] = None  # [max_seq, d/2, 2] float32 (llama)


def init_weights_compat(cfg: OracleConfig, seed: int, dtype=np.float64) -> OracleWeights:
    """One ``default_rng(seed)`` stream in the reference draw order
    (model.py:89-112): embed, then per layer wq wk wv wo w1 w2, then head."""
    cfg.validate()
    if not cfg.compat:
        raise OracleContractError("compat init needs the reference model family")
    rng = np.random.default_rng(seed)
    dt = np.dtype(dtype)
    h, f, v = cfg.hidden, cfg.ffn_dim, cfg.vocab_size

    def draw(*shape):
        return (rng.standard_normal(shape) * WEIGHT_SCALE).astype(dt)

    embed = draw(v, h)
    layers = []
    for _ in range(cfg.n_layers):
        lw = {}
        for name, shape in (("wq", (h, h)), ("wk", (h, h)), ("wv", (h, h)),
                            ("wo", (h, h)), ("w1", (h, f)), ("w2", (f, h))):
            lw[name] = draw(*shape)
        lw["attn_gain"] = np.ones(h, dtype=dt)
        lw["mlp_gain"] = np.ones(h, dtype=dt)
        layers.append(lw)
    return OracleWeights(cfg, dt, seed, embed, layers, np.ones(h, dtype=dt), draw(h, v))


# per-tensor stream tags for llama-mode init (independent draws per tensor)
_TAG_EMBED, _TAG_HEAD = 0, 1
_LAYER_TAGS = {"wq": 0, "wk": 1, "wv": 2, "wo": 3, "w_gate": 4, "w_up": 5, "w_down": 6,
               "w1": 4, "w2": 6}


def llama_tensor_shapes(cfg: OracleConfig) -> Dict[str, Tuple[int, int]]:
    h, d, f = cfg.hidden, cfg.head_dim, cfg.ffn_dim
    shapes = {"wq": (h, cfg.n_heads * d), "wk": (h, cfg.kv_heads * d),
              "wv": (h, cfg.kv_heads * d), "wo": (cfg.n_heads * d, h)}
    if cfg.mlp == "swiglu":
        shapes.update(w_gate=(h, f), w_up=(h, f), w_down=(f, h))
    else:
        shapes.update(w1=(h, f), w2=(f, h))
    return shapes


def draw_tensor(seed: int, tag: int, shape, bf16: bool) -> np.ndarray:
    """N(0, 0.02^2) from ``default_rng([seed, tag])``; float32 out."""
    x = np.random.default_rng([seed, tag]).standard_normal(shape, dtype=np.float32)
    x *= np.float32(WEIGHT_SCALE)
    return bf16_round(x) if bf16 else x


def init_weights_llama(cfg: OracleConfig, seed: int, dtype=np.float32,
                       bf16: bool = True) -> OracleWeights:
    """Per-tensor seeded streams; ``bf16=True`` rounds every matrix to
    bfloat16 so the oracle computes with exactly the GPU's weights."""
    cfg.validate()
    dt = np.dtype(dtype)
    h, v = cfg.hidden, cfg.vocab_size
    embed = draw_tensor(seed, _TAG_EMBED, (v, h), bf16).astype(dt)
    head = draw_tensor(seed, _TAG_HEAD, (h, v), bf16).astype(dt)
    layers = []
    for li in range(cfg.n_layers):
        lw = {}
        for name, shape in llama_tensor_shapes(cfg).items():
            tag = 16 + 16 * li + _LAYER_TAGS[name]
            lw[name] = draw_tensor(seed, tag, shape, bf16).astype(dt)
        lw["attn_gain"] = np.ones(h, dtype=dt)
        lw["mlp_gain"] = np.ones(h, dtype=dt)
        layers.append(lw)
    rope = None
    if cfg.pos == "rope":
        rope = rope_tables(cfg.max_seq, cfg.head_dim, cfg.rope_theta, cfg.rope_scaling)
    return OracleWeights(cfg, dt, seed, embed, layers, np.ones(h, dtype=dt), head, rope)


def partition_heads(n_heads: int, world_size: int) -> Tuple[Tuple[int, int], ...]:
    """Device d owns heads [d*H/P, (d+1)*H/P) (model.py:186-193)."""
    if world_size < 1 or n_heads % world_size:
        raise OracleContractError(f"{n_heads} heads do not split over {world_size}")
    w = n_heads // world_size
    return tuple((r * w, (r + 1) * w) for r in range(world_size))


def greedy_token(logits: np.ndarray) -> int:
    """Argmax; lowest index wins ties (model.py:303-307)."""
    if logits.ndim != 1:
        raise OracleContractError("greedy_token wants one row")
    return int(np.argmax(logits))


class Rounder:
    """Optional bf16 rounding at the points where the GPU stores bf16."""

    def __init__(self, on: bool):
        self.on = on

    def __call__(self, x: np.ndarray) -> np.ndarray:
        return bf16_round(x).astype(x.dtype) if self.on else x


def embed_rows(w: OracleWeights, toks: np.ndarray, positions: np.ndarray) -> np.ndarray:
    """x = E[tok] (+ sinusoidal positions in compat mode, model.py:342)."""
    x = w.embed[toks]
    if w.config.pos == "sinusoidal":
        x = x + sinusoidal_positions(positions, w.config.hidden, dtype=w.dtype)
    return x


def qkv_heads(w: OracleWeights, lw: dict, xn: np.ndarray, positions, rnd: Rounder,
              cols: Optional[Tuple[slice, slice]] = None, meter=None):
    """q [n, Hq, d], k/v [n, Hkv, d] after positions; ``cols`` selects a TP
    column block (q-slice, kv-slice)."""
    cfg = w.config
    d, n = cfg.head_dim, xn.shape[0]
    wq, wk, wv = lw["wq"], lw["wk"], lw["wv"]
    if cols is not None:
        qs, ks = cols
        wq, wk, wv = wq[:, qs], wk[:, ks], wv[:, ks]
    q = rnd(matmul(xn, wq, meter)).reshape(n, wq.shape[1] // d, d)
    k = rnd(matmul(xn, wk, meter)).reshape(n, wk.shape[1] // d, d)
    v = rnd(matmul(xn, wv, meter)).reshape(n, wv.shape[1] // d, d)
    if cfg.pos == "rope":
        q = rnd(rope_apply(q, positions, w.rope))
        k = rnd(rope_apply(k, positions, w.rope))
    return q, k, v


def mlp_block(w: OracleWeights, lw: dict, xn2: np.ndarray, rnd: Rounder,
              fcols: Optional[slice] = None, meter=None) -> np.ndarray:
    """gelu(xn·W1)·W2 (model.py:351) or down(silu(xn·Wg) * (xn·Wu))."""
    sl = slice(None) if fcols is None else fcols
    if w.config.mlp == "gelu":
        hid = gelu(matmul(xn2, lw["w1"][:, sl], meter))
        return matmul(hid, lw["w2"][sl, :], meter)
    g = matmul(xn2, lw["w_gate"][:, sl], meter)
    u = matmul(xn2, lw["w_up"][:, sl], meter)
    return matmul(rnd(silu(g) * u), lw["w_down"][sl, :], meter)


def forward_reference(w: OracleWeights, tokens: Sequence[int],
                      cache: Optional[OracleKvCache] = None,
                      emulate_bf16: bool = False):
    """Single-device forward over new tokens, continuing an optional cache.

    model.py:310-354.  Returns (logits [n, V], cache).
    """
    cfg = w.config
    eps = cfg.norm_eps
    rnd = Rounder(emulate_bf16)
    toks = np.asarray(tokens, dtype=np.int64)
    if toks.ndim != 1 or toks.size == 0:
        raise OracleContractError("forward_reference wants a non-empty token list")
    if toks.min() < 0 or toks.max() >= cfg.vocab_size:
        raise OracleContractError("token id out of vocab range")
    if cache is None:
        cache = OracleKvCache(cfg.n_layers, ((0, cfg.kv_heads),), cfg.head_dim,
                              cfg.max_seq, w.dtype)
    t0 = cache.token_count
    n = toks.size
    pos = np.arange(t0, t0 + n)
    x = embed_rows(w, toks, pos)
    for li, lw in enumerate(w.layers):
        xn = rnd(rms_norm(x, lw["attn_gain"], eps))
        q, k, v = qkv_heads(w, lw, xn, pos, rnd)
        cache.append(0, li, k, v)
        att = np.empty((n, cfg.n_heads, cfg.head_dim), dtype=w.dtype)
        for hq in range(cfg.n_heads):
            kw, vw = cache.read_window(0, li, hq // cfg.group)
            att[:, hq, :] = attend_cached(q[:, hq, :], kw, vw, t0)
        x = x + matmul(rnd(att).reshape(n, cfg.hidden), lw["wo"])
        xn2 = rnd(rms_norm(x, lw["mlp_gain"], eps))
        x = x + mlp_block(w, lw, xn2, rnd)
    cache.commit(n)
    logits = matmul(rnd(rms_norm(x, w.final_gain, eps)), w.head)
    return logits, cache


def reference_greedy(w: OracleWeights, prompt: Sequence[int], steps: int,
                     emulate_bf16: bool = False) -> List[int]:
    """Greedy continuation with the dense forward (model.py:357-366)."""
    if steps <= 0:
        return []
    logits, cache = forward_reference(w, prompt, emulate_bf16=emulate_bf16)
    out = [greedy_token(logits[-1])]
    while len(out) < steps:
        logits, cache = forward_reference(w, [out[-1]], cache, emulate_bf16=emulate_bf16)
        out.append(greedy_token(logits[-1]))
    return out
