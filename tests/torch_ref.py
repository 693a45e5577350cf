"""Dense torch fp32 restatement of the oracle forward — TEST INFRASTRUCTURE ONLY.

The numpy oracle (``oracle/``) is pinned bit-exactly to the reference
(``/root/reference/pkg/src/shiftsim``) but runs on host cores, so it cannot
check the product at the BASELINE shapes (8B x 32 layers x 8K tokens, B=64 x
ctx-2K decode, 32K SwiftKV).  This module restates the same algorithm
op-for-op in torch so it can run on the GPU in fp32 (TF32 off):

* ``forward``         — ``oracle.model.forward_reference`` (reference
                        ``model.py:310-354``): embed (+ sinusoidal in compat
                        mode), pre-norm blocks, causal attention over the
                        window ``t0 + m`` (``tensor_core.py:135-176``), final
                        norm and head; the optional bf16 rounding points are the
                        oracle's ``Rounder`` ones;
* ``forward_swiftkv`` — the SwiftKV prefill of ``oracle.engine`` (reference
                        ``parallel_engine.py:400-450``): K/V of layers >= cut
                        projected from ``z = rms_norm(x_cut, gain_cut)``, only
                        each request's last row through layers >= cut.

The chain stays pinned: ``tests/test_torch_ref.py`` checks this module
against the numpy oracle on the CPU (fp32 and f64) before the GPU tests use it
as the checker.  Only ``tests/`` imports it; the product never does.
"""

from __future__ import annotations

import math
from typing import Callable, Dict, List, Optional, Sequence

import numpy as np
import torch
import torch.nn.functional as F


class RefConfig:
    def __init__(self, n_layers, n_heads, kv_heads, head_dim, ffn_dim, vocab_size, pos, mlp,
                 norm_eps):
        self.n_layers, self.n_heads, self.kv_heads = n_layers, n_heads, kv_heads
        self.head_dim, self.ffn_dim, self.vocab_size = head_dim, ffn_dim, vocab_size
        self.pos, self.mlp, self.norm_eps = pos, mlp, norm_eps

    @property
    def hidden(self) -> int:
        return self.n_heads * self.head_dim

    @property
    def group(self) -> int:
        return self.n_heads // self.kv_heads

    @classmethod
    def of(cls, c) -> "RefConfig":
        return cls(c.n_layers, c.n_heads, c.kv_heads, c.head_dim, c.ffn_dim, c.vocab_size, c.pos,
                   c.mlp, c.norm_eps)


class RefWeights:
    """Weights in nn.Linear orientation ([out, in]); ``layer(i)`` materialises
    one layer in the compute dtype on demand (8B fp32 = 32 GB never exists at
    once)."""

    def __init__(self, cfg: RefConfig, device, dtype, embed, head, final_gain,
                 layer_fn: Callable[[int], Dict[str, torch.Tensor]], rope=None, pos_table=None):
        self.cfg, self.device, self.dtype = cfg, torch.device(device), dtype
        self.embed, self.head, self.final_gain = embed, head, final_gain
        self._layer_fn = layer_fn
        self.rope, self.pos_table = rope, pos_table
        self._memo: Optional[Dict[int, Dict[str, torch.Tensor]]] = None

    def keep_layers(self) -> "RefWeights":
        """Materialise each layer once and keep it (many short forwards)."""
        self._memo = {}
        return self

    def layer(self, i: int) -> Dict[str, torch.Tensor]:
        if self._memo is not None and i in self._memo:
            return self._memo[i]
        out = {k: v.to(self.dtype).contiguous() for k, v in self._layer_fn(i).items()}
        if self._memo is not None:
            self._memo[i] = out
        return out

    # ------------------------------------------------------------ sources
    @classmethod
    def from_oracle(cls, ow, device="cpu", dtype=torch.float32) -> "RefWeights":
        """From ``oracle.OracleWeights`` ([in, out] numpy matrices)."""
        cfg = RefConfig.of(ow.config)
        dev = torch.device(device)

        def t(a, transpose=False):
            a = np.asarray(a)
            return torch.as_tensor(np.ascontiguousarray(a.T if transpose else a), device=dev)

        names = ("wq", "wk", "wv", "wo") + (("w_gate", "w_up", "w_down") if cfg.mlp == "swiglu"
                                             else ("w1", "w2"))

        def layer_fn(i):
            lw = ow.layers[i]
            out = {n: t(lw[n], transpose=True) for n in names}
            out["attn_gain"] = t(lw["attn_gain"])
            out["mlp_gain"] = t(lw["mlp_gain"])
            return out

        rope = None if ow.rope is None else torch.as_tensor(ow.rope, device=dev)
        return cls(cfg, dev, dtype, t(ow.embed).to(dtype), t(ow.head, transpose=True).to(dtype),
                   t(ow.final_gain).to(dtype), layer_fn, rope=rope)

    @classmethod
    def from_model(cls, mw, dtype=torch.float32) -> "RefWeights":
        """From the product's device ``ModelWeights``: undo the fused/permuted
        layouts (per-rank q|k|v rows, gate/up interleave) — the bf16 VALUES are
        the ones the kernels read, upcast per layer."""
        from paper_2507_11830_b200.weights import ModelWeights

        c = mw.config
        cfg = RefConfig.of(c)
        dev = mw.embed.device
        d = c.head_dim
        idx = torch.as_tensor(ModelWeights._qkv_rows(c, mw.world_size), device=dev)
        nq, nk = c.n_heads * d, c.kv_heads * d

        def layer_fn(i):
            lw = mw.layers[i]
            qkv = torch.empty_like(lw.wqkv)
            qkv[idx] = lw.wqkv
            out = {"wq": qkv[:nq], "wk": qkv[nq:nq + nk], "wv": qkv[nq + nk:], "wo": lw.wo,
                   "attn_gain": lw.attn_gain, "mlp_gain": lw.mlp_gain}
            if c.mlp == "swiglu":
                f, h = c.ffn_dim, c.hidden
                v = lw.wgu.view(f // 128, 2, 128, h)
                out.update(w_gate=v[:, 0].reshape(f, h), w_up=v[:, 1].reshape(f, h),
                           w_down=lw.wdown)
            else:
                out.update(w1=lw.wgu, w2=lw.wdown)
            return out

        return cls(cfg, dev, dtype, mw.embed, mw.head, mw.final_gain, layer_fn, rope=mw.rope,
                   pos_table=mw.pos_table)


# ------------------------------------------------------------------ primitives
def _rnd(on: bool):
    return (lambda x: x.to(torch.bfloat16).to(x.dtype)) if on else (lambda x: x)


def rms_norm(x: torch.Tensor, gain: torch.Tensor, eps: float) -> torch.Tensor:
    """tensor_core.py:115-123 (eps typed like x)."""
    ms = (x * x).mean(dim=-1, keepdim=True)
    return gain * (x / torch.sqrt(ms + eps))


def gelu(x: torch.Tensor) -> torch.Tensor:
    """tensor_core.py:126-132, tanh form."""
    c = math.sqrt(2.0 / math.pi)
    return 0.5 * x * (1.0 + torch.tanh(c * (x + 0.044715 * x * x * x)))


def rope_apply(x: torch.Tensor, pos: torch.Tensor, table: torch.Tensor) -> torch.Tensor:
    """Rotate-half RoPE on x [n, heads, d] (oracle.prims.rope_apply)."""
    half = x.shape[-1] // 2
    cs = table[pos.long()].to(x.dtype)  # [n, half, 2]
    c, s = cs[:, None, :, 0], cs[:, None, :, 1]
    lo, hi = x[..., :half], x[..., half:]
    return torch.cat([lo * c - hi * s, hi * c + lo * s], dim=-1)


def sinusoidal(pos: torch.Tensor, width: int, dtype) -> torch.Tensor:
    """tensor_core.py:184-206 (f64, then cast)."""
    p = pos.to(torch.float64)[:, None]
    i = torch.arange(width // 2, dtype=torch.float64, device=pos.device)
    ang = p * torch.pow(torch.tensor(10000.0, dtype=torch.float64), -2.0 * i / width)[None]
    out = torch.empty((pos.shape[0], width), dtype=torch.float64, device=pos.device)
    out[:, 0::2] = torch.sin(ang)
    out[:, 1::2] = torch.cos(ang)
    return out.to(dtype)


def attend(q: torch.Tensor, K: torch.Tensor, V: torch.Tensor, t0: int,
           budget: int = 1 << 30, round_p: bool = False) -> torch.Tensor:
    """Causal GQA attention (tensor_core.py:135-176 per head): q [m, Hq, d]
    at positions t0.., K/V [T, Hkv, d] with T == t0 + m; query chunks keep the
    score tensor under ``budget`` elements.  ``round_p`` stores the
    unnormalised probabilities exp(s - max) as bf16 before P·V and divides
    by their f32 sum afterwards — where a flash-attention kernel keeps P in
    bf16 for the tensor-core P·V (the GPU's TMEM/register P tile)."""
    m, hq, d = q.shape
    T, hk, _ = K.shape
    if t0 + m != T:
        raise ValueError(f"attend window {t0}+{m} != {T}")
    g = hq // hk
    scale = 1.0 / math.sqrt(d)
    Kh, Vh = K.permute(1, 0, 2), V.permute(1, 0, 2)   # [Hkv, T, d]
    out = torch.empty_like(q)
    chunk = max(1, budget // max(1, hq * T))
    for lo in range(0, m, chunk):
        hi = min(m, lo + chunk)
        c, w = hi - lo, t0 + hi                        # keys beyond the chunk's last query are masked
        qc = q[lo:hi].permute(1, 0, 2).reshape(hk, g * c, d)
        s = torch.bmm(qc, Kh[:, :w].transpose(1, 2)).mul_(scale).view(hk, g, c, w)
        qpos = t0 + lo + torch.arange(c, device=q.device)
        vis = torch.arange(w, device=q.device)[None, :] <= qpos[:, None]
        s.masked_fill_(~vis, float("-inf"))
        if round_p:
            e = torch.exp(s - s.amax(dim=-1, keepdim=True))
            denom = e.sum(dim=-1, keepdim=True)
            e = e.to(torch.bfloat16).to(e.dtype)
            o = (torch.bmm(e.view(hk, g * c, w), Vh[:, :w]).view(hk, g, c, d) / denom).view(hq, c, d)
            out[lo:hi] = o.permute(1, 0, 2)
            del s, e
            continue
        p = torch.softmax(s, dim=-1).view(hk, g * c, w)
        o = torch.bmm(p, Vh[:, :w]).view(hq, c, d)
        out[lo:hi] = o.permute(1, 0, 2)
        del s, p
    return out


class RefCache:
    """Dense per-layer K/V [T, Hkv, d] in the compute dtype."""

    def __init__(self, n_layers: int):
        self.k: List[Optional[torch.Tensor]] = [None] * n_layers
        self.v: List[Optional[torch.Tensor]] = [None] * n_layers
        self.token_count = 0

    def append(self, layer: int, k: torch.Tensor, v: torch.Tensor) -> None:
        self.k[layer] = k if self.k[layer] is None else torch.cat([self.k[layer], k])
        self.v[layer] = v if self.v[layer] is None else torch.cat([self.v[layer], v])


def _qkv(rw, lw, xn, pos, rnd):
    cfg = rw.cfg
    n, d = xn.shape[0], cfg.head_dim
    q = rnd(xn @ lw["wq"].T).view(n, cfg.n_heads, d)
    k = rnd(xn @ lw["wk"].T).view(n, cfg.kv_heads, d)
    v = rnd(xn @ lw["wv"].T).view(n, cfg.kv_heads, d)
    if cfg.pos == "rope":
        q = rnd(rope_apply(q, pos, rw.rope))
        k = rnd(rope_apply(k, pos, rw.rope))
    return q, k, v


def _mlp(rw, lw, xn2, rnd):
    if rw.cfg.mlp == "gelu":
        return gelu(xn2 @ lw["w1"].T) @ lw["w2"].T
    g = xn2 @ lw["w_gate"].T
    u = xn2 @ lw["w_up"].T
    return rnd(F.silu(g) * u) @ lw["w_down"].T


def _embed(rw, toks, pos):
    x = rw.embed[toks.long()].to(rw.dtype)
    if rw.cfg.pos == "sinusoidal":
        x = x + sinusoidal(pos, rw.cfg.hidden, rw.dtype)
    return x


@torch.no_grad()
def forward(rw: RefWeights, tokens: Sequence[int], cache: Optional[RefCache] = None,
            emulate_bf16: bool = False, logit_rows: Optional[Sequence[int]] = None,
            hidden_out: Optional[dict] = None, round_p: bool = False):
    """oracle.forward_reference in torch.  Returns (logits [rows, V], cache);
    ``logit_rows`` selects the rows whose logits are computed (default all).
    ``hidden_out``, if given, receives the final-norm input rows.
    ``emulate_bf16`` rounds at the oracle's Rounder points; ``round_p`` also
    keeps attention probabilities in bf16 (see ``attend``)."""
    cfg, dev = rw.cfg, rw.device
    rnd = _rnd(emulate_bf16)
    eps = cfg.norm_eps
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        toks = torch.as_tensor(np.asarray(tokens, dtype=np.int64), device=dev)
        cache = RefCache(cfg.n_layers) if cache is None else cache
        t0, n = cache.token_count, toks.shape[0]
        pos = torch.arange(t0, t0 + n, device=dev)
        x = _embed(rw, toks, pos)
        for li in range(cfg.n_layers):
            lw = rw.layer(li)
            xn = rnd(rms_norm(x, lw["attn_gain"], eps))
            q, k, v = _qkv(rw, lw, xn, pos, rnd)
            cache.append(li, k, v)
            att = attend(q, cache.k[li], cache.v[li], t0, round_p=round_p)
            x = x + rnd(att).reshape(n, cfg.hidden) @ lw["wo"].T
            xn2 = rnd(rms_norm(x, lw["mlp_gain"], eps))
            x = x + _mlp(rw, lw, xn2, rnd)
            del lw
        cache.token_count += n
        rows = x if logit_rows is None else x[torch.as_tensor(list(logit_rows), dtype=torch.long,
                                                              device=dev)]
        if hidden_out is not None:
            hidden_out["x"] = rows
        if rows.shape[0] == 0:
            return rows.new_zeros((0, cfg.vocab_size)), cache
        logits = rnd(rms_norm(rows, rw.final_gain.to(rw.dtype), eps)) @ rw.head.to(rw.dtype).T
        return logits, cache
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old


@torch.no_grad()
def forward_swiftkv(rw: RefWeights, tokens: Sequence[int], cut: int,
                    emulate_bf16: bool = False, round_p: bool = False):
    """SwiftKV prefill of one request (oracle engine ``_tail_tp``, reference
    parallel_engine.py:400-450).  Returns (last-row logits [1, V], cache)."""
    cfg, dev = rw.cfg, rw.device
    rnd = _rnd(emulate_bf16)
    eps = cfg.norm_eps
    old = torch.backends.cuda.matmul.allow_tf32
    torch.backends.cuda.matmul.allow_tf32 = False
    try:
        toks = torch.as_tensor(np.asarray(tokens, dtype=np.int64), device=dev)
        cache = RefCache(cfg.n_layers)
        n, d = toks.shape[0], cfg.head_dim
        pos = torch.arange(n, device=dev)
        x = _embed(rw, toks, pos)
        for li in range(cut):
            lw = rw.layer(li)
            xn = rnd(rms_norm(x, lw["attn_gain"], eps))
            q, k, v = _qkv(rw, lw, xn, pos, rnd)
            cache.append(li, k, v)
            att = attend(q, k, v, 0, round_p=round_p)
            x = x + rnd(att).reshape(n, cfg.hidden) @ lw["wo"].T
            xn2 = rnd(rms_norm(x, lw["mlp_gain"], eps))
            x = x + _mlp(rw, lw, xn2, rnd)
        z = rnd(rms_norm(x, rw.layer(cut)["attn_gain"], eps))
        for li in range(cut, cfg.n_layers):
            lw = rw.layer(li)
            k = rnd(z @ lw["wk"].T).view(n, cfg.kv_heads, d)
            v = rnd(z @ lw["wv"].T).view(n, cfg.kv_heads, d)
            if cfg.pos == "rope":
                k = rnd(rope_apply(k, pos, rw.rope))
            cache.append(li, k, v)
        xt = x[n - 1:n]
        tpos = pos[n - 1:n]
        for li in range(cut, cfg.n_layers):
            lw = rw.layer(li)
            xn = rnd(rms_norm(xt, lw["attn_gain"], eps))
            q = rnd(xn @ lw["wq"].T).view(1, cfg.n_heads, d)
            if cfg.pos == "rope":
                q = rnd(rope_apply(q, tpos, rw.rope))
            att = attend(q, cache.k[li], cache.v[li], n - 1, round_p=round_p)
            xt = xt + rnd(att).reshape(1, cfg.hidden) @ lw["wo"].T
            xn2 = rnd(rms_norm(xt, lw["mlp_gain"], eps))
            xt = xt + _mlp(rw, lw, xn2, rnd)
        cache.token_count = n
        logits = rnd(rms_norm(xt, rw.final_gain.to(rw.dtype), eps)) @ rw.head.to(rw.dtype).T
        return logits, cache
    finally:
        torch.backends.cuda.matmul.allow_tf32 = old
