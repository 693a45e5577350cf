"""Dense CPU primitives of the oracle (test infrastructure only).

Compat-mode functions restate ``/root/reference/pkg/src/shiftsim/tensor_core.py``
operation-for-operation so that results are bit-identical to the reference:

* ``matmul``               — tensor_core.py:75-102 (ascending-k einsum; the
                             single-column case uses an explicit loop, :94-99)
* ``softmax_rows``         — tensor_core.py:105-112
* ``rms_norm``             — tensor_core.py:115-123
* ``gelu``                 — tensor_core.py:126-132
* ``attend_cached``        — tensor_core.py:135-176
* ``sinusoidal_positions`` — tensor_core.py:184-206

Llama-mode additions (not expressible in the reference):
``silu``, ``rope_tables`` / ``rope_apply`` (rotate-half RoPE, Llama-3.1
"llama3" frequency scaling) and ``bf16_round`` (round-to-nearest-even to
bfloat16, used to give the oracle the exact weights the GPU holds).
"""

from __future__ import annotations

import math
from typing import Optional, Sequence

import numpy as np

_OK_DTYPES = (np.dtype(np.float32), np.dtype(np.float64))


class OracleContractError(ValueError):
    """Raised when an oracle primitive is called outside its contract."""


def _finite(arr: np.ndarray, what: str) -> np.ndarray:
    # tensor_core.py:61-64 — every op checks its result for NaN/Inf
    if not np.all(np.isfinite(arr)):
        raise OracleContractError(f"{what}: non-finite result")
    return arr


def matmul(a: np.ndarray, b: np.ndarray, meter=None) -> np.ndarray:
    """c[i,j] = sum_t a[i,t] b[t,j], accumulated in ascending t.

    Follows tensor_core.py:75-102: operands are made C-contiguous, a
    single-column right operand is reduced by an explicit ascending loop
    (numpy's one-column kernel reorders partial sums), everything else goes
    through ``np.einsum(..., optimize=False)``.
    """
    if a.ndim != 2 or b.ndim != 2:
        raise OracleContractError(f"matmul wants 2-d operands: {a.shape} {b.shape}")
    if a.dtype not in _OK_DTYPES or a.dtype != b.dtype:
        raise OracleContractError(f"matmul dtypes {a.dtype}/{b.dtype}")
    if a.shape[1] != b.shape[0] or a.shape[1] == 0:
        raise OracleContractError(f"matmul inner dims {a.shape} x {b.shape}")
    lhs = np.ascontiguousarray(a)
    rhs = np.ascontiguousarray(b)
    if meter is not None:
        meter.add_matmul(lhs.shape[0], lhs.shape[1], rhs.shape[1])
    if rhs.shape[1] == 1 and rhs.shape[0] > 1:
        acc = np.zeros((lhs.shape[0], 1), dtype=lhs.dtype)
        for t in range(rhs.shape[0]):
            acc[:, 0] += lhs[:, t] * rhs[t, 0]
        return _finite(acc, "matmul")
    return _finite(np.einsum("ik,kj->ij", lhs, rhs, optimize=False), "matmul")


def softmax_rows(x: np.ndarray) -> np.ndarray:
    """Shift-by-max softmax over the last axis (tensor_core.py:105-112)."""
    top = np.max(x, axis=-1, keepdims=True)
    ex = np.exp(x - top)
    return _finite(ex / np.sum(ex, axis=-1, keepdims=True), "softmax_rows")


def rms_norm(x: np.ndarray, gain: np.ndarray, eps: float = 1e-6) -> np.ndarray:
    """gain * x / sqrt(mean(x^2) + eps) per row (tensor_core.py:115-123)."""
    if gain.shape != x.shape[-1:]:
        raise OracleContractError("rms_norm gain width mismatch")
    ms = np.mean(x * x, axis=-1, keepdims=True)
    den = np.sqrt(ms + x.dtype.type(eps))
    return _finite(gain * (x / den), "rms_norm")


def gelu(x: np.ndarray) -> np.ndarray:
    """tanh-form GeLU with dtype-typed constants (tensor_core.py:126-132)."""
    t = x.dtype.type
    c, k = t(math.sqrt(2.0 / math.pi)), t(0.044715)
    return _finite(t(0.5) * x * (t(1.0) + np.tanh(c * (x + k * x * x * x))), "gelu")


def silu(x: np.ndarray) -> np.ndarray:
    """x * sigmoid(x) — the Llama SwiGLU gate activation."""
    t = x.dtype.type
    return _finite(x / (t(1.0) + np.exp(-x)), "silu")


def attend_cached(q: np.ndarray, keys: np.ndarray, values: np.ndarray,
                  first_query_pos: int, meter=None) -> np.ndarray:
    """Causal single-head attention of q rows against a key window.

    tensor_core.py:135-176: query row i sits at absolute position
    ``first_query_pos + i`` and may see keys ``j <= first_query_pos + i``; the
    window must end exactly at the last query (T == first_query_pos + m).
    """
    m, d = q.shape
    t = keys.shape[0]
    if m < 1 or keys.shape != values.shape or keys.shape[1] != d:
        raise OracleContractError("attend_cached shape contract")
    if first_query_pos < 0 or first_query_pos + m != t:
        raise OracleContractError(f"attend_cached window {first_query_pos}+{m}!={t}")
    scale = q.dtype.type(1.0 / math.sqrt(d))
    s = matmul(q, np.ascontiguousarray(keys.T), meter=meter) * scale
    visible = np.arange(t)[None, :] <= (first_query_pos + np.arange(m)[:, None])
    s = np.where(visible, s, q.dtype.type(-np.inf))
    return matmul(softmax_rows(s), values, meter=meter)


def sinusoidal_positions(positions: Sequence[int], width: int,
                         dtype: Optional[np.dtype] = None) -> np.ndarray:
    """row[2i]=sin(p/10000^(2i/w)), row[2i+1]=cos(...), f64 then cast
    (tensor_core.py:184-206)."""
    if width % 2:
        raise OracleContractError("sinusoidal width must be even")
    p = np.asarray(positions, dtype=np.float64)
    i = np.arange(width // 2, dtype=np.float64)
    ang = p[:, None] * np.power(10000.0, -2.0 * i / width)[None, :]
    out = np.empty((p.shape[0], width), dtype=np.float64)
    out[:, 0::2] = np.sin(ang)
    out[:, 1::2] = np.cos(ang)
    return out if dtype is None else out.astype(dtype)


# ---------------------------------------------------------------- llama mode

def llama3_inv_freq(head_dim: int, theta: float, scaling: Optional[dict]) -> np.ndarray:
    """Per-pair inverse frequencies (f64), with Llama-3.1 "llama3" scaling.

    The scaling follows the published Llama-3.1 recipe (factor, low/high
    frequency factors, original context): long wavelengths are divided by
    ``factor``, short ones kept, the band in between interpolated smoothly.
    """
    inv = 1.0 / np.power(float(theta), np.arange(0, head_dim, 2, dtype=np.float64) / head_dim)
    if not scaling:
        return inv
    factor = float(scaling["factor"])
    lo_f = float(scaling["low_freq_factor"])
    hi_f = float(scaling["high_freq_factor"])
    orig = float(scaling["original_max_position_embeddings"])
    wavelen = 2.0 * math.pi / inv
    lo_wl, hi_wl = orig / lo_f, orig / hi_f
    out = np.where(wavelen > lo_wl, inv / factor, inv)
    smooth = (orig / wavelen - lo_f) / (hi_f - lo_f)
    mid = (wavelen >= hi_wl) & (wavelen <= lo_wl)
    blended = (1.0 - smooth) * out / factor + smooth * out
    return np.where(mid, blended, out)


def rope_tables(max_pos: int, head_dim: int, theta: float,
                scaling: Optional[dict]) -> np.ndarray:
    """cos/sin table ``[max_pos, head_dim/2, 2]`` in float32.

    Angles are formed in f64 and rounded once; the GPU kernel reads exactly
    this table, so both sides rotate with identical coefficients.
    """
    inv = llama3_inv_freq(head_dim, theta, scaling)
    ang = np.arange(max_pos, dtype=np.float64)[:, None] * inv[None, :]
    tab = np.empty((max_pos, head_dim // 2, 2), dtype=np.float32)
    tab[..., 0] = np.cos(ang)
    tab[..., 1] = np.sin(ang)
    return tab


def rope_apply(x: np.ndarray, positions: np.ndarray, table: np.ndarray) -> np.ndarray:
    """Rotate-half RoPE on ``x[n, heads, d]`` at absolute ``positions[n]``.

    out[i] = x[i] cos - x[i+d/2] sin ; out[i+d/2] = x[i+d/2] cos + x[i] sin.
    """
    d = x.shape[-1]
    half = d // 2
    cs = table[np.asarray(positions, dtype=np.int64)].astype(x.dtype)  # [n, half, 2]
    c = cs[:, None, :, 0]
    s = cs[:, None, :, 1]
    lo, hi = x[..., :half], x[..., half:]
    out = np.empty_like(x)
    out[..., :half] = lo * c - hi * s
    out[..., half:] = hi * c + lo * s
    return out


def bf16_round(x: np.ndarray) -> np.ndarray:
    """Round float values to the nearest bfloat16 (ties to even); float32 out."""
    f = np.ascontiguousarray(x, dtype=np.float32)
    u = f.view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return u.astype(np.uint32).view(np.float32).reshape(f.shape)


def bf16_bits(x: np.ndarray) -> np.ndarray:
    """bfloat16 bit patterns (uint16) of ``bf16_round(x)``."""
    return (bf16_round(x).view(np.uint32) >> 16).astype(np.uint16)
