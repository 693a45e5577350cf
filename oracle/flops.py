"""Oracle FLOP mirror (test infrastructure only).

Restates ``/root/reference/pkg/src/shiftsim/flops.py``: ``shard_rows`` /
``shard_bounds`` (:68-80, contiguous split, remainder to the lowest ranks),
``FlopMeter`` (:23-32) and ``flop_count`` (:87-200), extended to GQA
(k/v projections are ``n_kv_heads * head_dim`` wide) and SwiGLU (gate + up +
down).  For the reference model family the numbers are identical.
"""

from __future__ import annotations

from typing import List, Optional, Sequence, Tuple


class FlopMeter:
    __slots__ = ("flops",)

    def __init__(self):
        self.flops = 0

    def add_matmul(self, m: int, k: int, n: int) -> None:
        self.flops += 2 * m * k * n


def shard_rows(total: int, world_size: int) -> List[int]:
    q, r = divmod(total, world_size)
    return [q + (1 if i < r else 0) for i in range(world_size)]


def shard_bounds(total: int, world_size: int) -> List[Tuple[int, int]]:
    out, lo = [], 0
    for n in shard_rows(total, world_size):
        out.append((lo, lo + n))
        lo += n
    return out


def _mm(m, k, n):
    return 2 * m * k * n


def flop_count(spans: Sequence[int], history: Sequence[int], mode: str, cfg, world_size: int,
               span_logits: bool = False, swiftkv_cut: Optional[int] = None) -> Tuple[int, ...]:
    """Per-device FLOPs of one pass (flops.py:87-200, GQA/SwiGLU-extended)."""
    p = world_size
    h, d, f, v = cfg.hidden, cfg.head_dim, cfg.ffn_dim, cfg.vocab_size
    qw, kvw = cfg.n_heads * d, cfg.kv_heads * d
    hq_l = cfg.n_heads // p
    n_mlp = 2 if cfg.mlp == "gelu" else 3
    big_m = sum(spans)
    wins = [t0 + m for m, t0 in zip(spans, history)]
    cut = swiftkv_cut if (swiftkv_cut is not None and swiftkv_cut < cfg.n_layers) else None
    n_full = cfg.n_layers if cut is None else cut
    n_req = len(spans)

    def attn(sp, ws):  # owned heads x all rows, full window (flops.py:116-117)
        return sum(hq_l * (_mm(m, d, w) + _mm(m, w, d)) for m, w in zip(sp, ws))

    def layer_cost(rows, width_div):
        return (_mm(rows, h, qw // width_div) + 2 * _mm(rows, h, kvw // width_div)
                + _mm(rows, qw // width_div, h) + n_mlp * _mm(rows, h, f // width_div))

    ends, acc = [], 0
    for m in spans:
        acc += m
        ends.append(acc - 1)
    per = [0] * p
    if mode == "tp":
        for r in range(p):
            per[r] += n_full * (layer_cost(big_m, p) + attn(spans, wins))
    else:
        rows = shard_rows(big_m, p)
        for r in range(p):
            per[r] += n_full * (layer_cost(rows[r], 1) + attn(spans, wins))
    bounds = shard_bounds(big_m, p)
    owned_ends = [sum(1 for e in ends if lo <= e < hi) for lo, hi in bounds]
    if cut is None:
        for r in range(p):
            if mode == "tp":
                per[r] += _mm(big_m if span_logits else n_req, h, v // p)
            else:
                cnt = (bounds[r][1] - bounds[r][0]) if span_logits else owned_ends[r]
                per[r] += _mm(cnt, h, v)
        return tuple(per)
    n_tail = cfg.n_layers - cut
    for r in range(p):
        if mode == "tp":
            proj = 2 * _mm(big_m, h, kvw // p)
            tail = layer_cost(n_req, p) - 2 * _mm(n_req, h, kvw // p) + attn([1] * n_req, wins)
            per[r] += n_tail * (proj + tail) + _mm(n_req, h, v // p)
        else:
            rows = shard_rows(big_m, p)
            proj = 2 * _mm(rows[r], h, kvw)
            tr = owned_ends[r]
            tail = layer_cost(tr, 1) - 2 * _mm(tr, h, kvw) + attn([1] * n_req, wins)
            per[r] += n_tail * (proj + tail) + _mm(tr, h, v)
    return tuple(per)
