"""Operator-level drop-in for the reference's primitive API on the B200 kernels.

Mirrors ``/root/reference/pkg/src/shiftsim/tensor_core.py`` name for name —
same arguments, shape / dtype / window contracts, meter charges and error
type (``ContractViolation``, raised before any device work) — with every
arithmetic op a libshiftpar.so kernel:

===================================  ==========  =================================
reference (tensor_core.py)           lines       device op
===================================  ==========  =================================
``matmul(a, b, meter)``              :75-102     ``sp_gemm_bf16`` (ordered regime)
``softmax_rows(x)``                  :105-112    ``sp_softmax_rows_f32``
``rms_norm(x, gain, eps)``           :115-123    ``sp_rms_norm_f32``
``gelu(x)``                          :126-132    ``sp_gelu_f32``
``attend_cached(q, keys, values,     :135-176    ``sp_attention`` over a one-head
first_query_pos, meter)``                        paged pool (tcgen05 / mma.sync)
``causal_attention(q, k, v, meter)`` :179-181    ``attend_cached(q, k, v, 0)``
``sinusoidal_positions(...)``        :184-206    host table builder (f64, as the
                                                 reference; data, not compute)
===================================  ==========  =================================

Numerics: matmul and attention operands are rounded to bf16 and accumulate in
f32 (tensor cores); norms, GeLU and softmax run in f32.  Results come back in
the caller's container and dtype (numpy f32/f64 -> numpy, torch -> torch), so
a reference caller runs unchanged and agrees with the f64 reference within the
bf16 tolerance the product states (2e-2), not bit-for-bit.  The reference's
ordering contract for ``matmul`` (column splits of ``b`` and row splits of
``a`` recombine bit-exactly, tensor_core.py:1-23) still holds: the drop-in
pins the GEMM's ordered regime (one ascending-K chain of 16-deep MMA steps per
output, the same K loop for every tile shape, never split-K), so TP column
shards and SP row shards of one projection give identical bits — the property
``check_kv_invariance`` (verify_checks.py:109-135) asserts.

``install(shiftsim)`` binds these into an imported reference package (the
binding a maintainer adds, INTEGRATION.md Level 2); tests/test_dropin_gpu.py
runs the reference's own ``Engine`` and invariant checks through it.

There is no CPU fallback: without libshiftpar.so or a CUDA device every op
raises (``LibraryMissing`` / ``ContractViolation``).
"""

from __future__ import annotations

import enum
import math
from typing import Callable, Optional, Sequence

import numpy as np
import torch

from . import ops
from .errors import ContractViolation

_SUPPORTED = (np.dtype(np.float32), np.dtype(np.float64))
_Error = ContractViolation  # install() widens it to also be the caller's ContractViolation
_BLOCK = 64                  # key-page size of the one-head pools attend_cached builds


class Precision(enum.Enum):
    """Numeric width of the caller's arrays (tensor_core.py:43-58)."""

    F32 = "f32"
    F64 = "f64"

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.float32 if self is Precision.F32 else np.float64)

    @classmethod
    def parse(cls, name: str) -> "Precision":
        try:
            return cls(name)
        except ValueError:
            raise _Error(f"unknown precision {name!r}") from None


# ------------------------------------------------------------------ plumbing
def _dtype(x) -> np.dtype:
    if isinstance(x, torch.Tensor):
        return {torch.float32: np.dtype(np.float32), torch.float64: np.dtype(np.float64)}.get(
            x.dtype, np.dtype(object))
    return np.asarray(x).dtype


def _check_operand(x, op: str):
    if x.ndim != 2:
        raise _Error(f"{op} expects 2-d operands, got shape {tuple(x.shape)}")
    if _dtype(x) not in _SUPPORTED:
        raise _Error(f"{op} expects f32/f64 operands, got {x.dtype}")
    return x


def _device() -> torch.device:
    if not torch.cuda.is_available():
        raise _Error("tensor_core: no CUDA device (there is no CPU fallback)")
    return torch.device("cuda", torch.cuda.current_device())


def _to_dev(x, dtype=torch.float32) -> torch.Tensor:
    if isinstance(x, torch.Tensor):
        return x.to(device=_device(), dtype=dtype).contiguous()
    return torch.as_tensor(np.ascontiguousarray(x), device=_device()).to(dtype).contiguous()


def _back(t: torch.Tensor, like):
    """Device f32 result -> the caller's container and dtype."""
    if isinstance(like, torch.Tensor):
        return t.to(device=like.device, dtype=like.dtype)
    return t.cpu().numpy().astype(_dtype(like), copy=False)


def _finite(t: torch.Tensor, op: str) -> torch.Tensor:
    if t.numel() and not bool(torch.isfinite(t).all()):
        raise _Error(f"{op} produced non-finite values")
    return t


def _pad_cols(t: torch.Tensor, cols: int) -> torch.Tensor:
    if t.shape[1] == cols:
        return t
    out = torch.zeros((t.shape[0], cols), dtype=t.dtype, device=t.device)
    out[:, :t.shape[1]] = t
    return out


def _round_up(n: int, m: int) -> int:
    return -(-n // m) * m


# ---------------------------------------------------------------- primitives
def matmul(a, b, meter=None):
    """c[i][j] = sum_t a[i][t] b[t][j] (tensor_core.py:75-102) on the tcgen05
    GEMM: bf16 operands, f32 accumulation, ordered regime."""
    _check_operand(a, "matmul")
    _check_operand(b, "matmul")
    if a.shape[1] != b.shape[0]:
        raise _Error(f"matmul inner dims differ: {tuple(a.shape)} x {tuple(b.shape)}")
    if _dtype(a) != _dtype(b):
        raise _Error(f"matmul operands mix dtypes: {a.dtype} vs {b.dtype}")
    if a.shape[1] == 0:
        raise _Error("matmul requires a non-empty inner dimension")
    m, k = a.shape
    n = b.shape[1]
    if meter is not None:
        meter.add_matmul(m, k, n)
    if m == 0 or n == 0:
        return _back(torch.zeros((m, n), device=_device()), a)
    kp, np_ = _round_up(k, 8), _round_up(n, 32)
    A = _pad_cols(_to_dev(a, torch.bfloat16), kp)                       # [M, K]
    Bt = torch.zeros((np_, kp), dtype=torch.bfloat16, device=A.device)  # [N, K] (K-major)
    Bt[:n, :k] = _to_dev(b, torch.bfloat16).t()
    D = torch.empty((m, np_), dtype=torch.float32, device=A.device)
    ops.gemm(A, Bt, D, ops.EPI_STORE_F32, M=m, N=np_, K=kp, lda=kp, ldb=kp, ldd=np_, ordered=True)
    return _back(_finite(D[:, :n], "matmul"), a)


def softmax_rows(x):
    """Row softmax with shift-by-max; -inf entries give 0 (tensor_core.py:105-112)."""
    if _dtype(x) not in _SUPPORTED:
        raise _Error(f"softmax_rows expects f32/f64, got {x.dtype}")
    shape = tuple(x.shape)
    X = _to_dev(x).reshape(-1, shape[-1])
    out = torch.empty_like(X)
    if X.numel():
        ops.softmax_rows_f32(X, out)
    return _back(_finite(out, "softmax_rows").reshape(shape), x)


def rms_norm(x, gain, eps: float = 1e-6):
    """y = gain * x / sqrt(mean(x^2) + eps) per row over the last axis
    (tensor_core.py:115-123)."""
    if _dtype(x) not in _SUPPORTED:
        raise _Error(f"rms_norm expects f32/f64, got {x.dtype}")
    if tuple(gain.shape) != tuple(x.shape[-1:]):
        raise _Error(f"rms_norm gain shape {tuple(gain.shape)} != ({x.shape[-1]},)")
    shape = tuple(x.shape)
    X = _to_dev(x).reshape(-1, shape[-1])
    out = torch.empty_like(X)
    if X.numel():  # an SP rank may own no returned row (empty shard)
        ops.rms_norm_f32(X, _to_dev(gain), float(eps), out)
    return _back(_finite(out, "rms_norm").reshape(shape), x)


def gelu(x):
    """tanh-form GeLU, elementwise (tensor_core.py:126-132)."""
    if _dtype(x) not in _SUPPORTED:
        raise _Error(f"gelu expects f32/f64, got {x.dtype}")
    X = _to_dev(x)
    out = torch.empty_like(X)
    if X.numel():
        ops.gelu_f32(X, out)
    return _back(_finite(out, "gelu"), x)


def attend_cached(q, keys, values, first_query_pos: int, meter=None):
    """Single-head causal attention of q rows (absolute positions
    first_query_pos..) against the key window keys/values [T, d] with
    T == first_query_pos + m (tensor_core.py:135-176), on the paged attention
    kernels: the window is laid out as a one-head pool of 64-key pages with an
    identity block table.  head_dim is zero-padded to the kernels' 32/64/128
    and q pre-scaled so the kernel's 1/sqrt(d_pad) becomes 1/sqrt(d)."""
    _check_operand(q, "attend_cached")
    _check_operand(keys, "attend_cached")
    if q.shape[0] < 1:
        raise _Error("attend_cached needs at least one query row")
    if tuple(keys.shape) != tuple(values.shape):
        raise _Error("attend_cached key/value shapes differ")
    if q.shape[1] != keys.shape[1]:
        raise _Error("attend_cached head dims differ")
    if first_query_pos < 0:
        raise _Error("attend_cached first_query_pos must be >= 0")
    m, d = q.shape
    t = keys.shape[0]
    if first_query_pos + m != t:
        raise _Error(f"attend_cached window mismatch: {first_query_pos} + {m} != {t}")
    dp = next((c for c in (32, 64, 128) if d <= c), None)
    if dp is None:
        raise _Error(f"attend_cached: head_dim {d} > 128 is not covered by the device kernels")
    if meter is not None:  # the reference's two matmuls (:172, :176)
        meter.add_matmul(m, d, t)
        meter.add_matmul(m, t, d)
    dev = _device()
    n_blocks = -(-t // _BLOCK)
    Q = _to_dev(q)
    if dp != d:
        Q = Q * math.sqrt(dp / d)
    Q = _pad_cols(Q.to(torch.bfloat16), dp)
    kpool = torch.zeros((n_blocks, 1, _BLOCK, dp), dtype=torch.bfloat16, device=dev)
    vpool = torch.zeros_like(kpool)
    kpool.view(-1, dp)[:t, :d] = _to_dev(keys, torch.bfloat16)
    vpool.view(-1, dp)[:t, :d] = _to_dev(values, torch.bfloat16)
    meta = torch.tensor([0, m, first_query_pos, t] + list(range(n_blocks)), dtype=torch.int32,
                        device=dev)
    cu, first, kvlen, bt = meta[0:2], meta[2:3], meta[3:4], meta[4:].view(1, n_blocks)
    out = torch.empty((m, dp), dtype=torch.bfloat16, device=dev)
    if m == 1:
        ws_bytes = ops.attn_workspace_bytes(1, 1, dp, t)
        ws = torch.empty(max(ws_bytes, 16) // 4 + 4, dtype=torch.float32, device=dev)
        ops.attention(Q, kpool, vpool, bt, cu, first, kvlen, out, n_items=1, work=None, n_work=0,
                      max_q_len=1, max_kv_len=t, q_heads=1, kv_heads=1, head_dim=dp,
                      block_size=_BLOCK, ws=ws)
    else:
        tt = ops.attn_tile_tokens(1, 1, dp, _BLOCK)
        starts = sorted(range(0, m, tt), key=lambda s: -s)   # heaviest causal tiles first
        work = torch.tensor([v for s in starts for v in (0, s)], dtype=torch.int32, device=dev)
        ops.attention(Q, kpool, vpool, bt, cu, first, kvlen, out, n_items=1, work=work,
                      n_work=len(starts), max_q_len=m, max_kv_len=t, q_heads=1, kv_heads=1,
                      head_dim=dp, block_size=_BLOCK, ws=None)
    return _back(_finite(out[:, :d].float(), "attend_cached"), q)


def causal_attention(q, k, v, meter=None):
    """softmax(mask(q k^T / sqrt(d))) v, causal, single head (tensor_core.py:179-181)."""
    return attend_cached(q, k, v, 0, meter=meter)


def sinusoidal_positions(positions: Sequence[int], width: int, dtype: Optional[np.dtype] = None):
    """Additive sinusoidal rows (tensor_core.py:184-206): f64, cast at the end.
    A position-table builder (host data), like the product's own
    ``weights.sinusoidal_table``."""
    if width % 2 != 0:
        raise _Error("sinusoidal_positions needs an even width")
    pos = np.asarray(positions, dtype=np.float64)
    if pos.ndim != 1:
        raise _Error("positions must be a 1-d sequence")
    if pos.size and pos.min() < 0:
        raise _Error("positions must be >= 0")
    half = np.arange(width // 2, dtype=np.float64)
    ang = pos[:, None] * np.power(10000.0, -2.0 * half / width)[None, :]
    out = np.empty((pos.shape[0], width), dtype=np.float64)
    out[:, 0::2] = np.sin(ang)
    out[:, 1::2] = np.cos(ang)
    return out if dtype is None else out.astype(dtype)


# ------------------------------------------------------------------ binding
OPS = ("matmul", "softmax_rows", "rms_norm", "gelu", "attend_cached", "causal_attention")


def install(ref_pkg, modules: Sequence[str] = ("tensor_core", "model", "parallel_engine")) -> Callable[[], None]:
    """Bind the device primitives into an imported reference package: every
    ``modules`` member of ``ref_pkg`` that imported one of ``OPS`` gets ours
    (the reference modules do ``from .tensor_core import matmul, ...``, so
    each importing module is patched, not just tensor_core).  Errors raised
    by the device ops become instances of BOTH this package's and the
    reference's ``ContractViolation``.  Returns a function that restores the
    originals."""
    global _Error
    import importlib
    saved = []
    ref_err = getattr(importlib.import_module(ref_pkg.__name__ + ".errors"), "ContractViolation",
                      None)
    prev_err = _Error
    if ref_err is not None and not issubclass(_Error, ref_err):
        _Error = type("ContractViolation", (ContractViolation, ref_err), {})
    here = globals()
    for mod_name in modules:
        mod = importlib.import_module(f"{ref_pkg.__name__}.{mod_name}")
        for op in OPS:
            if hasattr(mod, op):
                saved.append((mod, op, getattr(mod, op)))
                setattr(mod, op, here[op])

    def restore() -> None:
        global _Error
        for mod, op, fn in reversed(saved):
            setattr(mod, op, fn)
        _Error = prev_err

    return restore
