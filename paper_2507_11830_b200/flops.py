"""FLOP accounting and SP token sharding.

``shard_rows`` / ``shard_bounds`` follow /root/reference/pkg/src/shiftsim/
flops.py:68-80 (contiguous split of the flattened batch, remainder to the
lowest ranks).  ``FlopMeter`` follows :23-32.  ``flop_count`` is the analytic
per-device mirror of what this engine executes (:87-200), extended to GQA and
SwiGLU; fused GEMMs (q|k|v, gate|up) count the same 2·m·k·n as the separate
reference matmuls they replace.  Attention is counted over the full window
(:116-117); ``causal_attention_flops`` gives the causal half used for the
roofline numerator.
"""

from __future__ import annotations

from dataclasses import dataclass
from typing import List, Optional, Sequence, Tuple


class FlopMeter:
    __slots__ = ("flops",)

    def __init__(self) -> None:
        self.flops = 0

    def add_matmul(self, m: int, k: int, n: int) -> None:
        self.flops += 2 * m * k * n


def shard_rows(total: int, world_size: int) -> List[int]:
    base, rem = divmod(total, world_size)
    return [base + (1 if r < rem else 0) for r in range(world_size)]


def shard_bounds(total: int, world_size: int) -> List[Tuple[int, int]]:
    out, lo = [], 0
    for n in shard_rows(total, world_size):
        out.append((lo, lo + n))
        lo += n
    return out


@dataclass(frozen=True)
class PassShape:
    spans: Tuple[int, ...]
    history: Tuple[int, ...]
    span_logits: bool = False

    @property
    def total_new_tokens(self) -> int:
        return sum(self.spans)


def _mm(m, k, n):
    return 2 * m * k * n


def flop_count(shape: PassShape, mode, cfg, world_size: int,
               swiftkv_cut: Optional[int] = None) -> Tuple[int, ...]:
    mode = getattr(mode, "value", mode)
    p = world_size
    h, d, f, v = cfg.hidden, cfg.head_dim, cfg.ffn_dim, cfg.vocab_size
    qw, kvw = cfg.n_heads * d, cfg.kv_heads * d
    hq = cfg.n_heads // p
    n_mlp = 3 if cfg.mlp == "swiglu" else 2
    spans, hist = shape.spans, shape.history
    big_m = sum(spans)
    wins = [t0 + m for m, t0 in zip(spans, hist)]
    cut = swiftkv_cut if (swiftkv_cut is not None and swiftkv_cut < cfg.n_layers) else None
    n_full = cfg.n_layers if cut is None else cut
    n_req = len(spans)

    def attn(sp, ws):
        return sum(hq * (_mm(m, d, w) + _mm(m, w, d)) for m, w in zip(sp, ws))

    def dense(rows, div):
        return (_mm(rows, h, (qw + 2 * kvw) // div) + _mm(rows, qw // div, h)
                + n_mlp * _mm(rows, h, f // div) + (0 if n_mlp == 2 else 0))

    ends, acc = [], 0
    for m in spans:
        acc += m
        ends.append(acc - 1)
    bounds = shard_bounds(big_m, p)
    owned = [sum(1 for e in ends if lo <= e < hi) for lo, hi in bounds]
    rows = shard_rows(big_m, p)
    per = [0] * p
    for r in range(p):
        if mode == "tp":
            per[r] += n_full * (dense(big_m, p) + attn(spans, wins))
        else:
            per[r] += n_full * (dense(rows[r], 1) + attn(spans, wins))
    if cut is None:
        for r in range(p):
            if mode == "tp":
                per[r] += _mm(big_m if shape.span_logits else n_req, h, v // p)
            else:
                per[r] += _mm(rows[r] if shape.span_logits else owned[r], h, v)
        return tuple(per)
    n_tail = cfg.n_layers - cut
    for r in range(p):
        if mode == "tp":
            proj = _mm(big_m, h, 2 * kvw // p)
            tail = (_mm(n_req, h, qw // p) + _mm(n_req, qw // p, h)
                    + n_mlp * _mm(n_req, h, f // p) + attn([1] * n_req, wins))
            per[r] += n_tail * (proj + tail) + _mm(n_req, h, v // p)
        else:
            proj = _mm(rows[r], h, 2 * kvw)
            tr = owned[r]
            tail = (_mm(tr, h, qw) + _mm(tr, qw, h) + n_mlp * _mm(tr, h, f)
                    + attn([1] * n_req, wins))
            per[r] += n_tail * (proj + tail) + _mm(tr, h, v)
    return tuple(per)


def causal_attention_flops(cfg, spans: Sequence[int], history: Sequence[int]) -> int:
    """4·d·H·Σ_i (t0+i+1) per layer, all layers — the causal half."""
    tot = 0
    for m, t0 in zip(spans, history):
        # sum_{i=0}^{m-1} (t0 + i + 1)
        tot += m * t0 + m * (m + 1) // 2
    return 4 * cfg.head_dim * cfg.n_heads * tot * cfg.n_layers


def gemm_flops_per_token(cfg) -> int:
    """2h(H+2Hkv)d + 2Hd·h + (2|3)·2h·f per layer, times layers."""
    h, d, f = cfg.hidden, cfg.head_dim, cfg.ffn_dim
    n_mlp = 3 if cfg.mlp == "swiglu" else 2
    per_layer = 2 * h * (cfg.n_heads + 2 * cfg.kv_heads) * d + 2 * cfg.n_heads * d * h \
        + n_mlp * 2 * h * f
    return per_layer * cfg.n_layers


def swiftkv_flop_ratio(cfg, prompt_len: int, cut_layer: Optional[int] = None) -> float:
    """Prefill FLOP ratio early-exit / standard (reference flops.py:203-215):
    one request of ``prompt_len`` tokens on one device (TP and SP coincide),
    ``cut_layer`` defaulting to the halfway cut."""
    cut = cfg.n_layers // 2 if cut_layer is None else cut_layer
    shape = PassShape(spans=(prompt_len,), history=(0,))
    early = sum(flop_count(shape, "tp", cfg, 1, swiftkv_cut=cut))
    std = sum(flop_count(shape, "tp", cfg, 1))
    return early / std

