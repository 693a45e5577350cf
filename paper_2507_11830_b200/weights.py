"""Device-resident bf16 weights in the layouts the sm_100a kernels consume.

The reference keeps f32/f64 ``x @ W`` matrices and materialises TP shards as
copies (model.py:220-254).  Here every GPU holds ONE bf16 replica (the SP
layout) and a TP shard is a zero-copy view of it (containment,
model.py:257-281):

* ``wqkv`` [P*W, h], W = (Hq/P + 2 Hkv/P) * d, rows grouped per rank r as
  [q heads of r | k heads of r | v heads of r].  SP multiplies by the whole
  matrix and its epilogue writes each rank's W columns straight into that
  peer's all-to-all send block; TP rank r multiplies by rows [rW, (r+1)W).
* ``wo`` [h, Hq*d] (nn.Linear [out, in]); TP rank r reads the K window of
  its heads through the GEMM's strided TMA map.
* ``wgu`` [2f, h], gate/up rows interleaved in 128-row chunks so a 256-wide
  N tile carries matching gate and up columns (SwiGLU epilogue); TP rank r
  owns the contiguous rows [r 2f/P, (r+1) 2f/P).  (GeLU mode: ``w1`` [f, h].)
* ``wdown`` [h, f]; TP uses the K window [r f/P, (r+1) f/P).
* ``head`` [V, h] (vocab rows; TP rank r owns rows [r V/P, (r+1) V/P)).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Dict, List, Optional

import numpy as np
import torch

from .config import ModelConfig
from .errors import ConfigError

WEIGHT_SCALE = 0.02  # reference model.py:86


def llama3_inv_freq(head_dim: int, theta: float, scaling: Optional[dict]) -> np.ndarray:
    """Rotary inverse frequencies (f64) with the published Llama-3.1 scaling."""
    inv = 1.0 / np.power(float(theta), np.arange(0, head_dim, 2, dtype=np.float64) / head_dim)
    if not scaling:
        return inv
    factor = float(scaling["factor"])
    lo, hi = float(scaling["low_freq_factor"]), float(scaling["high_freq_factor"])
    orig = float(scaling["original_max_position_embeddings"])
    wl = 2.0 * math.pi / inv
    scaled = np.where(wl > orig / lo, inv / factor, inv)
    t = (orig / wl - lo) / (hi - lo)
    band = (wl >= orig / hi) & (wl <= orig / lo)
    return np.where(band, (1.0 - t) * scaled / factor + t * scaled, scaled)


def rope_table(max_pos: int, head_dim: int, theta: float, scaling: Optional[dict]) -> np.ndarray:
    """cos/sin [max_pos, d/2, 2] f32 (angles in f64, rounded once)."""
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * llama3_inv_freq(head_dim, theta, scaling)[None]
    out = np.empty((max_pos, head_dim // 2, 2), dtype=np.float32)
    out[..., 0] = np.cos(ang)
    out[..., 1] = np.sin(ang)
    return out


def sinusoidal_table(max_pos: int, width: int) -> np.ndarray:
    """Additive sinusoidal rows (reference tensor_core.py:184-206), f64 -> f32."""
    i = np.arange(width // 2, dtype=np.float64)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * np.power(10000.0, -2.0 * i / width)[None]
    out = np.empty((max_pos, width), dtype=np.float64)
    out[:, 0::2] = np.sin(ang)
    out[:, 1::2] = np.cos(ang)
    return out.astype(np.float32)


@dataclass
class LayerWeights:
    wqkv: torch.Tensor
    wo: torch.Tensor
    wgu: torch.Tensor            # SwiGLU interleaved [2f, h] or GeLU w1 [f, h]
    wdown: torch.Tensor
    attn_gain: torch.Tensor
    mlp_gain: torch.Tensor
    wkv: Optional[torch.Tensor] = None   # SwiftKV: per-rank [k | v] rows [P*2*Hkv_l*d, h]


@dataclass
class ModelWeights:
    config: ModelConfig
    world_size: int
    embed: torch.Tensor
    layers: List[LayerWeights]
    final_gain: torch.Tensor
    head: torch.Tensor
    rope: Optional[torch.Tensor]
    pos_table: Optional[torch.Tensor]
    seed: Optional[int] = None

    # ---------------------------------------------------------- geometry
    @property
    def qkv_width(self) -> int:
        c, p = self.config, self.world_size
        return (c.n_heads // p + 2 * (c.kv_heads // p)) * c.head_dim

    def nbytes(self) -> int:
        n = self.embed.nbytes + self.head.nbytes
        for lw in self.layers:
            n += lw.wqkv.nbytes + lw.wo.nbytes + lw.wgu.nbytes + lw.wdown.nbytes
        return n

    # ------------------------------------------------------- construction
    @staticmethod
    def _qkv_rows(cfg: ModelConfig, p: int) -> np.ndarray:
        """Row order of the fused [q; k; v] (nn.Linear) matrix grouped per rank."""
        d = cfg.head_dim
        hq, hk = cfg.n_heads // p, cfg.kv_heads // p
        q0, k0, v0 = 0, cfg.n_heads * d, (cfg.n_heads + cfg.kv_heads) * d
        rows = []
        for r in range(p):
            rows.append(np.arange(q0 + r * hq * d, q0 + (r + 1) * hq * d))
            rows.append(np.arange(k0 + r * hk * d, k0 + (r + 1) * hk * d))
            rows.append(np.arange(v0 + r * hk * d, v0 + (r + 1) * hk * d))
        return np.concatenate(rows)

    @staticmethod
    def _kv_rows(cfg: ModelConfig, p: int) -> np.ndarray:
        d = cfg.head_dim
        hk = cfg.kv_heads // p
        k0, v0 = cfg.n_heads * d, (cfg.n_heads + cfg.kv_heads) * d
        rows = []
        for r in range(p):
            rows.append(np.arange(k0 + r * hk * d, k0 + (r + 1) * hk * d))
            rows.append(np.arange(v0 + r * hk * d, v0 + (r + 1) * hk * d))
        return np.concatenate(rows)

    @staticmethod
    def _interleave_gu(gate: torch.Tensor, up: torch.Tensor) -> torch.Tensor:
        f, h = gate.shape
        out = torch.empty((2 * f, h), dtype=gate.dtype, device=gate.device)
        v = out.view(f // 128, 2, 128, h)
        v[:, 0].copy_(gate.view(f // 128, 128, h))
        v[:, 1].copy_(up.view(f // 128, 128, h))
        return out

    @classmethod
    def _assemble(cls, cfg: ModelConfig, p: int, device, embed, head, final_gain, layer_fn,
                  seed=None) -> "ModelWeights":
        cfg.validate()
        cfg.check_world(p)
        qkv_idx = torch.as_tensor(cls._qkv_rows(cfg, p), device=device)
        layers = []
        for li in range(cfg.n_layers):
            t = layer_fn(li)  # dict of nn.Linear-oriented bf16 tensors on device
            fused = torch.cat([t["q"], t["k"], t["v"]], dim=0).index_select(0, qkv_idx).contiguous()
            if cfg.mlp == "swiglu":
                wgu = cls._interleave_gu(t["gate"], t["up"])
            else:
                wgu = t["w1"].contiguous()
            layers.append(LayerWeights(
                wqkv=fused, wo=t["o"].contiguous(), wgu=wgu, wdown=t["down"].contiguous(),
                attn_gain=t["attn_gain"].float().contiguous(),
                mlp_gain=t["mlp_gain"].float().contiguous()))
            del t
        rope = pos = None
        if cfg.pos == "rope":
            rope = torch.as_tensor(rope_table(cfg.max_seq, cfg.head_dim, cfg.rope_theta,
                                              cfg.rope_scaling), device=device)
        else:
            pos = torch.as_tensor(sinusoidal_table(cfg.max_seq, cfg.hidden), device=device)
        return cls(cfg, p, embed.contiguous(), layers, final_gain.float().contiguous(),
                   head.contiguous(), rope, pos, seed)

    @classmethod
    def from_host(cls, cfg: ModelConfig, host: Dict, world_size: int, device="cuda") -> "ModelWeights":
        """Upload reference-oriented host weights ([in, out] matrices, as in
        model.py:63-84) rounded to bf16."""
        dev = torch.device(device)

        def bf(x):  # [in, out] numpy -> nn.Linear [out, in] bf16 on device
            return torch.as_tensor(np.ascontiguousarray(np.asarray(x, dtype=np.float32).T),
                                   device=dev).to(torch.bfloat16)

        def layer_fn(li):
            lw = host["layers"][li]
            t = {"q": bf(lw["wq"]), "k": bf(lw["wk"]), "v": bf(lw["wv"]), "o": bf(lw["wo"]),
                 "attn_gain": torch.as_tensor(np.asarray(lw["attn_gain"], np.float32), device=dev),
                 "mlp_gain": torch.as_tensor(np.asarray(lw["mlp_gain"], np.float32), device=dev)}
            if cfg.mlp == "swiglu":
                t.update(gate=bf(lw["w_gate"]), up=bf(lw["w_up"]), down=bf(lw["w_down"]))
            else:
                t.update(w1=bf(lw["w1"]), down=bf(lw["w2"]))
            return t

        embed = torch.as_tensor(np.asarray(host["embed"], np.float32), device=dev).to(torch.bfloat16)
        head = bf(host["head"])
        gain = torch.as_tensor(np.asarray(host["final_gain"], np.float32), device=dev)
        return cls._assemble(cfg, world_size, dev, embed, head, gain, layer_fn, host.get("seed"))

    @classmethod
    def random(cls, cfg: ModelConfig, seed: int, world_size: int, device="cuda") -> "ModelWeights":
        """N(0, 0.02^2) bf16 weights drawn on the device (8B/70B bench init;
        the reference draws from one host stream, model.py:89-112)."""
        dev = torch.device(device)
        gen = torch.Generator(device=dev)
        gen.manual_seed(seed)
        h, d, f = cfg.hidden, cfg.head_dim, cfg.ffn_dim

        def draw(*shape):
            out = torch.empty(shape, dtype=torch.bfloat16, device=dev)
            flat = out.view(-1)
            step = 1 << 26
            for s in range(0, flat.numel(), step):
                n = min(step, flat.numel() - s)
                tmp = torch.randn(n, generator=gen, device=dev, dtype=torch.float32)
                flat[s:s + n].copy_(tmp.mul_(WEIGHT_SCALE))
            return out

        def layer_fn(li):
            t = {"q": draw(cfg.n_heads * d, h), "k": draw(cfg.kv_heads * d, h),
                 "v": draw(cfg.kv_heads * d, h), "o": draw(h, cfg.n_heads * d),
                 "attn_gain": torch.ones(h, device=dev), "mlp_gain": torch.ones(h, device=dev)}
            if cfg.mlp == "swiglu":
                t.update(gate=draw(f, h), up=draw(f, h), down=draw(h, f))
            else:
                t.update(w1=draw(f, h), down=draw(h, f))
            return t

        embed = draw(cfg.vocab_size, h)
        head = draw(cfg.vocab_size, h)
        return cls._assemble(cfg, world_size, dev, embed, head, torch.ones(h, device=dev),
                             layer_fn, seed)

    def ensure_swiftkv(self, cut: int) -> None:
        """Build the per-rank [k | v] projection rows for layers >= cut (SwiftKV)."""
        cfg, p = self.config, self.world_size
        fused_rows = self._qkv_rows(cfg, p)
        pos_of = np.empty_like(fused_rows)
        pos_of[fused_rows] = np.arange(fused_rows.size)
        idx = torch.as_tensor(pos_of[self._kv_rows(cfg, p)], device=self.embed.device)
        for li in range(cut, cfg.n_layers):
            lw = self.layers[li]
            if lw.wkv is None:
                lw.wkv = lw.wqkv.index_select(0, idx).contiguous()


# ------------------------------------------------- TP shards as views
@dataclass
class TpLayerShard:
    """One layer of a TP rank: zero-copy views of the resident replica."""

    wqkv: torch.Tensor    # rows [rW, (r+1)W) of the fused per-rank q|k|v matrix
    wo: torch.Tensor      # K window [:, r Hq/P d : (r+1) Hq/P d] (strided view)
    wgu: torch.Tensor     # rows of the rank's ffn shard (gate|up interleaved, or w1)
    wdown: torch.Tensor   # K window [:, r f/P : (r+1) f/P]


@dataclass
class TpShard:
    """What device ``rank`` reads under TP (reference model.py:206-217)."""

    rank: int
    world_size: int
    head_range: tuple
    kv_head_range: tuple
    vocab_range: tuple
    ffn_range: tuple
    layers: List[TpLayerShard]
    head_rows: torch.Tensor   # [V/P, h] vocab rows of the LM head


def tp_shard_view(weights: ModelWeights, rank: int, world_size: Optional[int] = None) -> TpShard:
    """The blocks device ``rank`` owns under TP (reference model.py:220-254),
    as views of the one bf16 replica — the same views the engine's TP pass
    multiplies by (the reference materialises copies)."""
    from .errors import ContractViolation
    cfg = weights.config
    p = weights.world_size if world_size is None else world_size
    if p != weights.world_size:
        raise ConfigError(f"weights are laid out for P={weights.world_size}, not {p}")
    if not 0 <= rank < p:
        raise ContractViolation(f"rank {rank} out of range for P={p}")
    d = cfg.head_dim
    hq, hk, fl, vs = cfg.n_heads // p, cfg.kv_heads // p, cfg.ffn_dim // p, cfg.vocab_size // p
    W = weights.qkv_width
    gu = 2 * fl if cfg.mlp == "swiglu" else fl
    layers = [TpLayerShard(wqkv=lw.wqkv[rank * W:(rank + 1) * W],
                           wo=lw.wo[:, rank * hq * d:(rank + 1) * hq * d],
                           wgu=lw.wgu[rank * gu:(rank + 1) * gu],
                           wdown=lw.wdown[:, rank * fl:(rank + 1) * fl])
              for lw in weights.layers]
    return TpShard(rank, p, (rank * hq, (rank + 1) * hq), (rank * hk, (rank + 1) * hk),
                   (rank * vs, (rank + 1) * vs), (rank * fl, (rank + 1) * fl), layers,
                   weights.head[rank * vs:(rank + 1) * vs])


def _inside(view: torch.Tensor, base: torch.Tensor) -> bool:
    """view's elements all live inside base's storage (same buffer, in range)."""
    if view.untyped_storage().data_ptr() != base.untyped_storage().data_ptr():
        return False
    lo = view.data_ptr()
    hi = lo + ((view.shape[0] - 1) * view.stride(0) + (view.shape[1] - 1) * view.stride(1) + 1) \
        * view.element_size()
    b_lo = base.data_ptr()
    return b_lo <= lo and hi <= b_lo + base.numel() * base.element_size()


def check_shard_containment(weights: ModelWeights, world_size: Optional[int] = None) -> bool:
    """Every element of every TP shard is a sub-block of the SP-resident
    replica (reference model.py:257-281).  Here containment holds by
    construction — a TP shard IS a view of the replica, no bytes are copied —
    and is checked structurally: each view aliases the replica's storage at
    the expected rows / columns."""
    cfg = weights.config
    p = weights.world_size if world_size is None else world_size
    d = cfg.head_dim
    for rank in range(p):
        sh = tp_shard_view(weights, rank, p)
        for lw, sl in zip(weights.layers, sh.layers):
            if not (_inside(sl.wqkv, lw.wqkv) and _inside(sl.wo, lw.wo)
                    and _inside(sl.wgu, lw.wgu) and _inside(sl.wdown, lw.wdown)):
                return False
            if sl.wo.shape[1] * p != lw.wo.shape[1] or sl.wqkv.shape[0] * p != lw.wqkv.shape[0]:
                return False
            if sl.wo.data_ptr() != lw.wo.data_ptr() + rank * (cfg.n_heads // p) * d * 2:
                return False
        if not _inside(sh.head_rows, weights.head):
            return False
    return True


def memory_report(config: ModelConfig, world_size: int) -> dict:
    """Parameter residency per device (reference model.py:284-300), for the
    GQA / SwiGLU geometry: matrix parameters shard exactly 1/P under TP; norm
    gains are replicated.  Shift parallelism keeps the SP replica resident, so
    ``replica_bytes_per_device`` (bf16) is what each GPU holds; the TP views a
    TP pass reads are 1/P of it.  Also the per-device KV bytes per token."""
    c = config
    h, f, v, L, d = c.hidden, c.ffn_dim, c.vocab_size, c.n_layers, c.head_dim
    n_mlp = 3 if c.mlp == "swiglu" else 2
    per_layer = h * (c.n_heads + 2 * c.kv_heads) * d + c.n_heads * d * h + n_mlp * h * f
    matrix = v * h + L * per_layer + h * v
    gains = L * 2 * h + h
    return {
        "matrix_params_total": matrix,
        "replicated_gain_params": gains,
        "sp_matrix_params_per_device": matrix,
        "tp_matrix_params_per_device": matrix // world_size,
        "sharded_ratio": world_size,
        "replica_bytes_per_device": 2 * matrix + 4 * gains,
        "tp_view_bytes_per_device": 2 * matrix // world_size,
        "kv_bytes_per_token_per_device": 2 * L * (c.kv_heads // world_size) * d * 2,
    }

