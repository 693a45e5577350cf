"""B200 cost model of one Shift-Parallel pass, and the SP<->TP crossover tau.

The reference decides the mode by batched-token count against
``default_token_threshold(P) = 4·P`` (parallel_engine.py:130-145) — a number
picked for its simulator.  On B200 the crossover follows from what differs
between the two modes for ONE rank of a P-GPU group at M new tokens:

* projections: the FLOPs per rank are identical (TP: M rows x 1/P of the
  weights; SP: M/P rows x the full replica), but SP streams P x the weight
  bytes, so SP only matches TP once its M/P rows make the GEMMs compute-bound
  (M/P >~ peak FLOP/s / HBM B/s ~ 200 rows on B200);
* collectives per layer: TP all-reduces M x h f32 partials twice (one-shot:
  (P-1) x M x h x 4 B read per rank; two-shot above
  ``two_shot_min_rows``: (P-1)/P x M x h x (4 + 2) B); SP exchanges
  (P-1)/P x M/P rows of q/k/v and of o in bf16 — ~P x fewer bytes;
* attention FLOPs and KV bytes are the same in both modes (each rank owns
  H/P heads over every token) and cancel.

``pass_us`` puts a roofline GEMM time (max of compute at the in-step tcgen05
rate and weight streaming, plus a per-launch cost — fitted to measured
per-rank timings, ``GemmModel``) next to the link model; ``crossover`` is the smallest M from
which SP stays at least as fast as TP.  The GEMM constants are calibrated
against tools/tau_sweep.py (per-layer projection times of one rank measured on
a B200 with the product's dispatch; profiles/r02_tau_sweep.json); the link
bandwidth is the pool's measured B200 peer copy (770 GB/s per direction), the
per-collective latency an estimate until a multi-GPU lease.
"""

from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache


@dataclass(frozen=True)
class LinkModel:
    nvlink_gbs: float = 770.0      # measured B200 peer copy per direction (B200_PROFILING.md)
    efficiency: float = 1.0        # fraction of that the fused peer stores / loads reach
    latency_us: float = 6.0        # per collective: flag handshake + launch (unmeasured)
    two_shot_min_rows: int = 256   # peer.two_shot_min_rows() default


@dataclass(frozen=True)
class GemmModel:
    """Least-squares fit (log error) to the 108 per-rank layer timings of
    tools/tau_sweep.py (profiles/r02_tau_sweep.json; 8B shapes, P = 2/4/8,
    M = 1..4096, graph-replayed): every GEMM costs max(compute, weight
    streaming) plus a fixed, non-overlapped ~9 us; the swap-AB regime
    (M <= 256 token rows, padded to 32; for projections wider than
    swap_wide_tiles 256-row weight tiles only up to swap_wide_max_rows, with
    one or more tiles per SM only up to swap_huge_max_rows, as
    gemm_tcgen05.cu:swap_regime) computes at ~800 TFLOP/s, the 128-row tiles
    above it at ~1400."""

    tflops: float = 1400.0         # 128/256-row tcgen05 tiles (M > swap_max_rows)
    swap_tflops: float = 800.0     # swap-AB regime
    swap_max_rows: int = 256
    swap_wide_max_rows: int = 64   # wide projections leave swap-AB above this
    swap_wide_tiles: int = 37      # "wide": more 256-row weight tiles than sms / 4
    swap_huge_tiles: int = 148     # at least one 256-row weight tile per SM ...
    swap_huge_max_rows: int = 32   # ... stays swap-AB only up to this many rows
    hbm_gbs: float = 6454.6        # MEASURED_PEAKS.json copy bandwidth
    stream_eff: float = 1.0        # weight streaming, fraction of hbm_gbs
    launch_us: float = 9.0         # per-GEMM fixed cost (launch, fill, drain, tail)


B200_LINKS = LinkModel()
B200_GEMM = GemmModel()


def _gemm_us(rows: int, n: int, k: int, g: GemmModel) -> float:
    if rows <= 0:
        return 0.0
    tiles = -(-n // 256)
    wide = tiles > g.swap_wide_tiles
    limit = g.swap_huge_max_rows if tiles >= g.swap_huge_tiles else (
        g.swap_wide_max_rows if wide else g.swap_max_rows)
    if rows <= limit:
        pad, tf = -(-rows // 32) * 32, g.swap_tflops
    else:
        pad, tf = -(-rows // 128) * 128, g.tflops
    compute = 2.0 * pad * n * k / (tf * 1e12)
    stream = (n * k + rows * k + rows * n) * 2.0 / (g.hbm_gbs * 1e9 * g.stream_eff)
    return max(compute, stream) * 1e6 + g.launch_us


def layer_gemm_us(cfg, mode: str, P: int, M: int, g: GemmModel = B200_GEMM) -> float:
    """One rank's four projections of one layer (QKV, O, gate/up, down)."""
    h, d, f = cfg.hidden, cfg.head_dim, cfg.ffn_dim
    W = (cfg.n_heads + 2 * cfg.kv_heads) * d
    up = 2 * f if cfg.mlp == "swiglu" else f
    if mode == "tp":
        rows, div = M, P
    else:
        rows, div = -(-M // P), 1
    return (_gemm_us(rows, W // div, h, g) + _gemm_us(rows, h, cfg.n_heads * d // div, g)
            + _gemm_us(rows, up // div, h, g) + _gemm_us(rows, h, f // div, g))


def comm_us(cfg, mode: str, P: int, M: int, links: LinkModel = B200_LINKS) -> float:
    """One layer's collectives for one rank (modelled; see module doc)."""
    if P <= 1:
        return 0.0
    bw = links.nvlink_gbs * 1e9 * links.efficiency
    h, d = cfg.hidden, cfg.head_dim
    if mode == "tp":
        if M <= links.two_shot_min_rows:
            per = (P - 1) * M * h * 4.0
        else:
            per = (P - 1) / P * M * h * (4.0 + 2.0)
        return 2 * (per / bw * 1e6 + links.latency_us)
    rows = -(-M // P)
    qkv = (P - 1) / P * rows * (cfg.n_heads + 2 * cfg.kv_heads) * d * 2.0
    o = (P - 1) / P * rows * cfg.n_heads * d * 2.0
    return (qkv + o) / bw * 1e6 + 2 * links.latency_us


def pass_us(cfg, mode: str, P: int, M: int, g: GemmModel = B200_GEMM,
            links: LinkModel = B200_LINKS) -> float:
    """Modelled per-rank time of the mode-dependent part of an M-token pass."""
    return cfg.n_layers * (layer_gemm_us(cfg, mode, P, M, g) + comm_us(cfg, mode, P, M, links))


@lru_cache(maxsize=64)
def _crossover(key, P: int, g: GemmModel, links: LinkModel) -> int:
    cfg = _Geom(*key)
    grid = sorted({*range(1, 65), *(int(2 ** (i / 8)) for i in range(48, 8 * 17))})
    sp_ok = [pass_us(cfg, "sp", P, m, g, links) <= pass_us(cfg, "tp", P, m, g, links) for m in grid]
    tau = grid[-1]
    for i in range(len(grid) - 1, -1, -1):
        if not sp_ok[i]:
            break
        tau = grid[i]
    return tau


@dataclass(frozen=True)
class _Geom:
    n_layers: int
    n_heads: int
    kv_heads: int
    head_dim: int
    ffn_dim: int
    mlp: str

    @property
    def hidden(self) -> int:
        return self.n_heads * self.head_dim


def crossover(cfg, P: int, g: GemmModel = B200_GEMM, links: LinkModel = B200_LINKS) -> int:
    """Smallest batched-token count from which SP is modelled no slower than TP."""
    if P <= 1:
        return 1
    key = (cfg.n_layers, cfg.n_heads, cfg.kv_heads, cfg.head_dim, cfg.ffn_dim, cfg.mlp)
    return _crossover(key, P, g, links)
