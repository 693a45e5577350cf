"""Typed wrappers over the C-ABI (include/shiftpar.h) for torch CUDA tensors.

Every wrapper validates its operands, forwards raw device pointers and the
current CUDA stream to libshiftpar.so, and maps a nonzero status to
``ContractViolation``.  ``kernel_launches()`` counts the kernels enqueued (the
``gpu_launches`` figure of bench.py): the C-side launch counter plus the kernel
nodes of replayed CUDA graphs.
"""

from __future__ import annotations

import ctypes
from typing import Optional

import torch

from . import _lib
from .errors import ContractViolation

EPI_STORE_BF16 = 0
EPI_STORE_F32 = 1
EPI_ADD_F32 = 2
EPI_SWIGLU = 3
EPI_GELU = 4
EPI_PARTIAL_F32 = 5  # raw K-split partials [n][M][N], n = gemm_partials(M, N, K)
GEMM_ORDERED = 0x100  # flag: one ascending-K chain per output (never split-K)

# Optional live per-kernel timing (bench.py roofline): when set to a dict, the
# wrapped launches record CUDA events on the launching stream plus their
# algorithmic work: PROFILE[kind] -> list of (start, end, flops, bytes).
PROFILE: Optional[dict] = None


class _Timed:
    def __init__(self, kind: str, flops: int = 0, nbytes: int = 0):
        self.kind, self.flops, self.nbytes = kind, flops, nbytes

    def __enter__(self):
        self.on = PROFILE is not None and not torch.cuda.is_current_stream_capturing()
        if self.on:
            self.ev = (torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
            self.ev[0].record()
        return self

    def __exit__(self, *exc):
        if self.on and exc[0] is None:
            self.ev[1].record()
            PROFILE.setdefault(self.kind, []).append((self.ev[0], self.ev[1], self.flops, self.nbytes))
        return False


_graph_launches = 0


def add_graph_launches(n: int) -> None:
    """Account kernels launched by a CUDA-graph replay (not seen by the C counter)."""
    global _graph_launches
    _graph_launches += n


def kernel_launches() -> int:
    """Kernels of libshiftpar.so launched in this process: counted in C for direct
    launches, plus the kernel nodes of every replayed CUDA graph."""
    return int(_lib.load().sp_kernel_launches()) + _graph_launches


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _ptr(t: Optional[torch.Tensor]) -> Optional[int]:
    return None if t is None else t.data_ptr()


def _need(t: torch.Tensor, dtype: torch.dtype, what: str) -> None:
    if not t.is_cuda:
        raise ContractViolation(f"{what}: tensor must live on the GPU")
    if t.dtype != dtype:
        raise ContractViolation(f"{what}: want {dtype}, got {t.dtype}")


def device_check() -> int:
    lib = _lib.load()
    n = ctypes.c_int(0)
    _lib.check(lib.sp_device_check(ctypes.byref(n)), "sp_device_check")
    return n.value


def gemm(a: torch.Tensor, b: torch.Tensor, d: torch.Tensor, epilogue: int, *, M: int, N: int,
         K: int, lda: int, ldb: int, ldd: int, a_kchunk: int = 0, a_chunk_stride: int = 0,
         peer_width: int = 0, peer_stride: int = 0, meter=None, ordered: bool = False) -> None:
    """D = epi(A[M,K] B[N,K]^T) — see sp_gemm_bf16.  A/B may be views with
    arbitrary base offsets (zero-copy TP shards).  ``ordered`` pins the
    one-chain-per-output regime (split-invariant at any M)."""
    _need(a, torch.bfloat16, "gemm A")
    _need(b, torch.bfloat16, "gemm B")
    if epilogue in (EPI_STORE_BF16, EPI_SWIGLU, EPI_GELU):
        _need(d, torch.bfloat16, "gemm D")
    else:
        _need(d, torch.float32, "gemm D")
    if epilogue == EPI_PARTIAL_F32 and d.numel() < gemm_partials(M, N, K) * M * N:
        raise ContractViolation("gemm: partial epilogue needs [gemm_partials(M,N,K), M, N] f32 D")
    if meter is not None:
        meter.add_matmul(M, K, N)
    if M == 0:
        return
    lib = _lib.load()
    nbytes = (M * K + N * K) * 2 + M * (N // 2 if epilogue == EPI_SWIGLU else N) * d.element_size()
    with _Timed("gemm", 2 * M * N * K, nbytes):  # (split-K reduce, if any, included)
        rc = lib.sp_gemm_bf16(a.data_ptr(), lda, a_kchunk, a_chunk_stride, b.data_ptr(), ldb,
                              d.data_ptr(), ldd, M, N, K,
                              epilogue | (GEMM_ORDERED if ordered else 0), peer_width,
                              peer_stride, _stream())
    _lib.check(rc, "sp_gemm_bf16")


def gemm_qkv_rope(a: torch.Tensor, b: torch.Tensor, *, M: int, K: int, lda: int, ldb: int,
                  pos: torch.Tensor, slot: torch.Tensor, rope: Optional[torch.Tensor],
                  q_out: Optional[torch.Tensor], k_pool: torch.Tensor, v_pool: torch.Tensor,
                  q_heads: int, kv_heads: int, block_size: int, meter=None) -> None:
    """QKV projection with RoPE + paged KV write in the epilogue (head_dim 128):
    bit-identical to gemm(EPI_STORE_BF16) followed by rope_kv_write."""
    _need(a, torch.bfloat16, "gemm A")
    _need(b, torch.bfloat16, "gemm B")
    N = (q_heads + 2 * kv_heads) * 128
    if meter is not None:
        meter.add_matmul(M, K, N)
    if M == 0:
        return
    nbytes = (M * K + N * K) * 2 + M * N * 2
    with _Timed("gemm", 2 * M * N * K, nbytes):
        rc = _lib.load().sp_gemm_bf16_qkv_rope(
            a.data_ptr(), lda, b.data_ptr(), ldb, M, K, pos.data_ptr(), slot.data_ptr(),
            _ptr(rope), _ptr(q_out), 0 if q_out is None else q_out.stride(0), k_pool.data_ptr(),
            v_pool.data_ptr(), q_heads, kv_heads, block_size, _stream())
    _lib.check(rc, "sp_gemm_bf16_qkv_rope")


GEMM_WS_BYTES = 64 << 20
# Every split-K workspace ever registered stays alive for the life of the
# process: captured CUDA graphs (decode passes) hold its raw address, so
# replacing it must never return the old buffer to the caching allocator
# (ADVICE r1).  One default buffer per device, shared by all engines on it
# (kernels on one stream run in order).
_ws_keep: list = []
_ws_default: dict = {}
_ws_current: dict = {}


def set_gemm_workspace(ws: Optional[torch.Tensor], device=None) -> None:
    """Register the split-K workspace of `ws`'s device (or `device` when ws is
    None: disables split-K there).  Registered buffers are never freed."""
    dev = torch.device(ws.device if ws is not None else (device or "cuda"))
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    nbytes = 0 if ws is None else ws.numel() * ws.element_size()
    if ws is not None:
        _ws_keep.append(ws)
    with torch.cuda.device(idx):
        _lib.check(_lib.load().sp_gemm_set_workspace(_ptr(ws), nbytes), "sp_gemm_set_workspace")
    _ws_current[idx] = None if ws is None else ws.data_ptr()


def ensure_gemm_workspace(device) -> torch.Tensor:
    """The device's default split-K workspace, allocated once and (re)registered
    if something else is registered there."""
    dev = torch.device(device)
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    ws = _ws_default.get(idx)
    if ws is None:
        ws = torch.empty(GEMM_WS_BYTES, dtype=torch.uint8, device=torch.device("cuda", idx))
        _ws_default[idx] = ws
    if _ws_current.get(idx) != ws.data_ptr():
        set_gemm_workspace(ws)
    return ws


def gemm_to_peers(a: torch.Tensor, b: torch.Tensor, peer_ptrs: torch.Tensor, *, row_off: int,
                  M: int, N: int, K: int, lda: int, ldb: int, ldd: int, peer_width: int,
                  epilogue: int = EPI_STORE_BF16, a_kchunk: int = 0, a_chunk_stride: int = 0,
                  peer_ptrs_host=None, meter=None) -> None:
    """GEMM whose epilogue stores column block n // peer_width of row m straight
    into peer_ptrs[block] at row row_off + m (fused seq->head all-to-all).
    ``peer_ptrs_host`` (the same pointers as a host int64 array) enables the
    TMA-store epilogue of the prefill regime."""
    _need(a, torch.bfloat16, "gemm A")
    _need(b, torch.bfloat16, "gemm B")
    if meter is not None:
        meter.add_matmul(M, K, N)
    if M == 0:
        return
    with _Timed("gemm", 2 * M * N * K, (M * K + N * K) * 2 + M * N * 2):
        host = None
        if peer_ptrs_host is not None:
            host = peer_ptrs_host.ctypes.data if hasattr(peer_ptrs_host, "ctypes") else \
                peer_ptrs_host.data_ptr()
        rc = _lib.load().sp_gemm_bf16_to_peers(a.data_ptr(), lda, a_kchunk, a_chunk_stride,
                                               b.data_ptr(), ldb, peer_ptrs.data_ptr(), host,
                                               row_off, ldd, M, N, K, epilogue, peer_width,
                                               _stream())
    _lib.check(rc, "sp_gemm_bf16_to_peers")


def peer_scatter_rows(src: torch.Tensor, rows_total: int, peers: int, my_rank: int,
                      dst_ptrs: torch.Tensor) -> None:
    """Row t of src goes to its SP owner's [P][rows_s][w] buffer (head->seq)."""
    if rows_total == 0:
        return
    _lib.check(_lib.load().sp_peer_scatter_rows(src.data_ptr(), src.stride(0), rows_total,
                                                src.shape[1], peers, my_rank, dst_ptrs.data_ptr(),
                                                _stream()), "sp_peer_scatter_rows")


def peer_signal(flag_ptrs: torch.Tensor, peers: int, my_rank: int) -> None:
    _lib.check(_lib.load().sp_peer_signal(flag_ptrs.data_ptr(), peers, my_rank, _stream()),
               "sp_peer_signal")


def peer_wait(flags: torch.Tensor, peers: int) -> None:
    _lib.check(_lib.load().sp_peer_wait(flags.data_ptr(), peers, _stream()), "sp_peer_wait")


def peer_allreduce_add_rmsnorm(part_ptrs: torch.Tensor, peers: int, x: torch.Tensor,
                               gain: Optional[torch.Tensor], eps: float,
                               out: Optional[torch.Tensor], rows: int, slabs: int = 1) -> None:
    """x += sum of the P peer partials (ascending rank; each rank's partial is
    its `slabs` K-split slabs [slabs][rows][h] summed first), then optional
    RMSNorm."""
    if rows == 0:
        return
    _lib.check(_lib.load().sp_peer_allreduce_add_rmsnorm(
        part_ptrs.data_ptr(), peers, slabs, x.data_ptr(), x.stride(0), _ptr(gain), float(eps),
        _ptr(out), 0 if out is None else out.stride(0), rows, x.shape[1], _stream()),
        "sp_peer_allreduce_add_rmsnorm")


def peer_reduce_scatter_rmsnorm(part_ptrs: torch.Tensor, peers: int, my_rank: int,
                                x: torch.Tensor, gain: torch.Tensor, eps: float,
                                xn_ptrs: torch.Tensor, ldo: int, rows: int) -> None:
    """Two-shot TP all-reduce: sum my row slice's P partials (ascending rank),
    add into x, push bf16 RMSNorm rows into every rank's xn buffer."""
    if rows == 0:
        return
    _lib.check(_lib.load().sp_peer_reduce_scatter_rmsnorm(
        part_ptrs.data_ptr(), peers, my_rank, x.data_ptr(), x.stride(0), gain.data_ptr(),
        float(eps), xn_ptrs.data_ptr(), ldo, rows, x.shape[1], _stream()),
        "sp_peer_reduce_scatter_rmsnorm")


def gather_rows_bf16(src: torch.Tensor, idx: torch.Tensor, dst: torch.Tensor) -> None:
    """dst[r] = src[idx[r]] for bf16 rows (16-byte vectors)."""
    _need(src, torch.bfloat16, "gather src")
    _need(dst, torch.bfloat16, "gather dst")
    rows = idx.shape[0]
    if rows == 0:
        return
    _lib.check(_lib.load().sp_gather_rows_bf16(src.data_ptr(), src.stride(0), idx.data_ptr(),
                                               dst.data_ptr(), dst.stride(0), rows, src.shape[1],
                                               _stream()), "sp_gather_rows_bf16")


def embed(ids: torch.Tensor, table: torch.Tensor, out: torch.Tensor,
          pos: Optional[torch.Tensor] = None, pos_table: Optional[torch.Tensor] = None) -> None:
    _need(ids, torch.int32, "embed ids")
    _need(table, torch.bfloat16, "embed table")
    _need(out, torch.float32, "embed out")
    rows = ids.shape[0]
    if rows == 0:
        return
    rc = _lib.load().sp_embed(ids.data_ptr(), table.data_ptr(), _ptr(pos), _ptr(pos_table),
                              out.data_ptr(), rows, table.shape[1], _stream())
    _lib.check(rc, "sp_embed")


def ipc_export(t: torch.Tensor) -> tuple:
    """(64-byte CUDA IPC handle of the allocation holding t, offset of t in it)."""
    h = ctypes.create_string_buffer(64)
    off = ctypes.c_int64(0)
    _lib.check(_lib.load().sp_ipc_export(t.data_ptr(), h, ctypes.byref(off)), "sp_ipc_export")
    return h.raw, off.value


def ipc_import(handle: bytes, offset: int) -> int:
    """Device address (in this process) of a peer's exported buffer."""
    ptr = ctypes.c_void_p(0)
    _lib.check(_lib.load().sp_ipc_import(ctypes.create_string_buffer(handle, 64), offset,
                                         ctypes.byref(ptr)), "sp_ipc_import")
    return int(ptr.value)


def gemm_partials(M: int, N: int, K: int) -> int:
    """How many f32 [M, N] partial slabs an EPI_PARTIAL_F32 GEMM writes."""
    return int(_lib.load().sp_gemm_partials(M, N, K))


def add_rmsnorm(x: torch.Tensor, gain: torch.Tensor, eps: float, out: torch.Tensor, *,
                add: Optional[torch.Tensor] = None, row_idx: Optional[torch.Tensor] = None,
                rows: Optional[int] = None, n_add: int = 1) -> None:
    """out = bf16(rms_norm(x (+)= sum of n_add [rows, h] slabs of `add`))."""
    _need(x, torch.float32, "rmsnorm x")
    _need(gain, torch.float32, "rmsnorm gain")
    _need(out, torch.bfloat16, "rmsnorm out")
    n = (row_idx.shape[0] if row_idx is not None else x.shape[0]) if rows is None else rows
    if n == 0:
        return
    h = x.shape[1]
    if add is not None:
        _need(add, torch.float32, "rmsnorm add")
        if add.numel() < n_add * n * h:
            raise ContractViolation("add_rmsnorm: add holds fewer than n_add [rows, h] slabs")
    rc = _lib.load().sp_add_rmsnorm(x.data_ptr(), x.stride(0), _ptr(add), n_add, gain.data_ptr(),
                                    float(eps), _ptr(row_idx), out.data_ptr(), out.stride(0), n, h,
                                    _stream())
    _lib.check(rc, "sp_add_rmsnorm")


def rope_kv_write(qkv: torch.Tensor, pos: torch.Tensor, slot: torch.Tensor,
                  rope: Optional[torch.Tensor], q_out: Optional[torch.Tensor],
                  k_pool: torch.Tensor, v_pool: torch.Tensor, *, rows: int, q_heads: int,
                  kv_heads: int, head_dim: int, block_size: int) -> None:
    _need(qkv, torch.bfloat16, "rope qkv")
    if rows == 0:
        return
    rc = _lib.load().sp_rope_kv_write(qkv.data_ptr(), qkv.stride(0), pos.data_ptr(),
                                      slot.data_ptr(), _ptr(rope), _ptr(q_out),
                                      0 if q_out is None else q_out.stride(0),
                                      k_pool.data_ptr(), v_pool.data_ptr(), rows, q_heads,
                                      kv_heads, head_dim, block_size, _stream())
    _lib.check(rc, "sp_rope_kv_write")


def rope_kv_write_partials(parts: torch.Tensor, n_parts: int, pos: torch.Tensor,
                           slot: torch.Tensor, rope: Optional[torch.Tensor],
                           q_out: Optional[torch.Tensor], k_pool: torch.Tensor,
                           v_pool: torch.Tensor, *, rows: int, q_heads: int, kv_heads: int,
                           head_dim: int, block_size: int) -> None:
    """rope_kv_write on a QKV projection left as n_parts K-split partials [n, rows, W]."""
    _need(parts, torch.float32, "rope partials")
    if rows == 0:
        return
    width = (q_heads + 2 * kv_heads) * head_dim
    if parts.numel() < n_parts * rows * width:
        raise ContractViolation("rope_kv_write_partials: parts smaller than [n, rows, W]")
    rc = _lib.load().sp_rope_kv_write_partials(
        parts.data_ptr(), n_parts, width, pos.data_ptr(), slot.data_ptr(), _ptr(rope),
        _ptr(q_out), 0 if q_out is None else q_out.stride(0), k_pool.data_ptr(),
        v_pool.data_ptr(), rows, q_heads, kv_heads, head_dim, block_size, _stream())
    _lib.check(rc, "sp_rope_kv_write_partials")


DL_RES_NORM = 0
DL_SWIGLU = 1
DL_ROPE_KV = 2


class DlProj:
    """One projection of a fused decode layer (sp_dl_proj): acc = x · w^T then
    ``kind`` (DL_RES_NORM: x_res += acc, out = norm · gain; DL_SWIGLU: out =
    silu(gate) · up; DL_ROPE_KV: q / paged K,V)."""

    def __init__(self, w: torch.Tensor, x: torch.Tensor, kind: int, *, n: int, k: int,
                 ldw: int, gain: Optional[torch.Tensor] = None,
                 out: Optional[torch.Tensor] = None):
        _need(w, torch.bfloat16, "decode_layer weight")
        _need(x, torch.bfloat16, "decode_layer input rows")
        if out is not None:
            _need(out, torch.bfloat16, "decode_layer output")
        self.w, self.x, self.kind, self.n, self.k, self.ldw = w, x, kind, n, k, ldw
        self.gain, self.out = gain, out


def _dl_args(rows, x, eps, projs, lead_gain, lead_out, rope_args, ws, sync):
    a = _lib.DecodeLayerArgs()
    a.rows, a.hidden = rows, x.shape[1]
    a.x, a.ldx, a.eps = x.data_ptr(), x.stride(0), eps
    a.n_proj = len(projs)
    for i, p in enumerate(projs):
        d = a.proj[i]
        d.w, d.ldw, d.x, d.ldx = p.w.data_ptr(), p.ldw, p.x.data_ptr(), p.x.stride(0)
        d.n, d.k, d.kind = p.n, p.k, p.kind
        d.gain = _ptr(p.gain)
        d.out = _ptr(p.out)
        d.ldo = 0 if p.out is None else p.out.stride(0)
    if lead_out is not None:
        a.lead_gain, a.lead_out, a.ld_lead = lead_gain.data_ptr(), lead_out.data_ptr(), lead_out.stride(0)
    if rope_args is not None:
        r = rope_args
        a.pos, a.slot, a.rope = r["pos"].data_ptr(), r["slot"].data_ptr(), _ptr(r["rope"])
        a.q_out, a.ldq = r["q_out"].data_ptr(), r["q_out"].stride(0)
        a.k_pool, a.v_pool = r["k_pool"].data_ptr(), r["v_pool"].data_ptr()
        a.q_heads, a.kv_heads = r["q_heads"], r["kv_heads"]
        a.block_size, a.head_dim = r["block_size"], r["head_dim"]
    if ws is not None:
        a.ws, a.ws_bytes = ws.data_ptr(), ws.numel() * ws.element_size()
    if sync is not None:
        a.sync = sync.data_ptr()
    return a


def decode_layer_ws_bytes(rows: int, x: torch.Tensor, projs) -> int:
    a = _dl_args(rows, x, 0.0, projs, None, None, None, None, None)
    n = int(_lib.load().sp_decode_layer_ws_bytes(ctypes.byref(a)))
    if n < 0:
        raise ContractViolation("decode_layer_ws_bytes: bad arguments")
    return n


def decode_layer(rows: int, x: torch.Tensor, eps: float, projs, *, ws: torch.Tensor,
                 sync: torch.Tensor, lead_gain: Optional[torch.Tensor] = None,
                 lead_out: Optional[torch.Tensor] = None, rope_args: Optional[dict] = None,
                 meter=None) -> None:
    """sp_decode_layer: the projections of one TP (P = 1) decode layer as ONE
    persistent kernel (see include/shiftpar.h).  ``sync``: 2 zeroed int32 owned
    by the caller (the kernel re-arms them)."""
    _need(x, torch.float32, "decode_layer residual")
    _need(sync, torch.int32, "decode_layer sync")
    if meter is not None:
        for p in projs:
            meter.add_matmul(rows, p.k, p.n)
    if rows == 0:
        return
    a = _dl_args(rows, x, eps, projs, lead_gain, lead_out, rope_args, ws, sync)
    flops = sum(2 * rows * p.n * p.k for p in projs)
    nbytes = sum(p.n * p.k * 2 for p in projs)
    with _Timed("decode_layer", flops, nbytes):
        rc = _lib.load().sp_decode_layer(ctypes.byref(a), _stream())
    _lib.check(rc, "sp_decode_layer")


def attn_tile_tokens(q_heads: int, kv_heads: int, head_dim: int, block_size: int) -> int:
    return _lib.load().sp_attn_tile_tokens(q_heads, kv_heads, head_dim, block_size)


def attn_workspace_bytes(n_items: int, q_heads: int, head_dim: int, max_kv: int) -> int:
    return _lib.load().sp_attn_workspace_bytes(n_items, q_heads, head_dim, max_kv)


def attention(q: torch.Tensor, k_pool: torch.Tensor, v_pool: torch.Tensor,
              block_tables: torch.Tensor, cu_q: torch.Tensor, first_pos: torch.Tensor,
              kv_len: torch.Tensor, out: torch.Tensor, *, n_items: int,
              work: Optional[torch.Tensor], n_work: int, max_q_len: int, max_kv_len: int,
              q_heads: int, kv_heads: int, head_dim: int, block_size: int,
              ws: Optional[torch.Tensor], work_flops: int = 0, work_bytes: int = 0) -> None:
    _need(q, torch.bfloat16, "attention q")
    _need(out, torch.bfloat16, "attention out")
    if n_items == 0:
        return
    ws_bytes = 0 if ws is None else ws.numel() * ws.element_size()
    kind = "attn_prefill" if n_work > 0 else "attn_decode"
    with _Timed(kind, work_flops, work_bytes):
        rc = _lib.load().sp_attention(q.data_ptr(), q.stride(0), q.shape[0], k_pool.data_ptr(),
                                      v_pool.data_ptr(), k_pool.shape[0],
                                      block_tables.data_ptr(), block_tables.stride(0),
                                      cu_q.data_ptr(), first_pos.data_ptr(), kv_len.data_ptr(),
                                      n_items, _ptr(work), n_work, max_q_len, max_kv_len,
                                      out.data_ptr(), out.stride(0), q_heads, kv_heads, head_dim,
                                      block_size, _ptr(ws), ws_bytes, _stream())
    _lib.check(rc, "sp_attention")


def attention_decode_qkv(parts: torch.Tensor, n_parts: int, pos: torch.Tensor,
                         slot: torch.Tensor, rope: Optional[torch.Tensor], k_pool: torch.Tensor,
                         v_pool: torch.Tensor, block_tables: torch.Tensor, cu_q: torch.Tensor,
                         kv_len: torch.Tensor, out: torch.Tensor, *, n_items: int,
                         max_kv_len: int, q_heads: int, kv_heads: int, block_size: int,
                         ws: Optional[torch.Tensor], work_flops: int = 0,
                         work_bytes: int = 0) -> None:
    """Decode attention fed by the QKV K-split partials [n_parts, rows, W]
    (sp_attention_decode_qkv): RoPE + the new token's KV write happen inside
    the attention kernel; bit-identical to rope_kv_write_partials + attention."""
    _need(parts, torch.float32, "attention_decode_qkv partials")
    _need(out, torch.bfloat16, "attention out")
    if n_items == 0:
        return
    width = (q_heads + 2 * kv_heads) * 128
    rows = parts.numel() // max(1, n_parts * width)
    if parts.numel() < n_parts * rows * width or rows < n_items:
        raise ContractViolation("attention_decode_qkv: parts smaller than [n, rows, W]")
    ws_bytes = 0 if ws is None else ws.numel() * ws.element_size()
    with _Timed("attn_decode", work_flops, work_bytes):
        rc = _lib.load().sp_attention_decode_qkv(
            parts.data_ptr(), n_parts, width, rows, pos.data_ptr(), slot.data_ptr(), _ptr(rope),
            k_pool.data_ptr(), v_pool.data_ptr(), k_pool.shape[0], block_tables.data_ptr(),
            block_tables.stride(0), cu_q.data_ptr(), kv_len.data_ptr(), n_items, max_kv_len,
            out.data_ptr(), out.stride(0), q_heads, kv_heads, block_size, _ptr(ws), ws_bytes,
            _stream())
    _lib.check(rc, "sp_attention_decode_qkv")


SPLIT_SLOT_BYTES = 256 * 130 * 4  # one (work entry, kv head) partial: O [256][128] + (m, l)


def attention_prefill_split(q, k_pool, v_pool, block_tables, cu_q, first_pos, kv_len, out, *,
                            work, split, n_work, combine, n_combine, n_slots, q_heads, kv_heads,
                            head_dim, block_size, ws, work_flops: int = 0,
                            work_bytes: int = 0) -> None:
    """Split-KV tcgen05 prefill (sp_attention_prefill_split); ws must hold
    n_slots * kv_heads partial slots."""
    _need(q, torch.bfloat16, "attention q")
    _need(out, torch.bfloat16, "attention out")
    need = n_slots * kv_heads * SPLIT_SLOT_BYTES
    if ws is None or ws.numel() * ws.element_size() < need:
        raise ContractViolation("attention split: workspace too small")
    with _Timed("attn_prefill", work_flops, work_bytes):
        rc = _lib.load().sp_attention_prefill_split(
            q.data_ptr(), q.stride(0), q.shape[0], k_pool.data_ptr(), v_pool.data_ptr(),
            k_pool.shape[0], block_tables.data_ptr(), block_tables.stride(0), cu_q.data_ptr(),
            first_pos.data_ptr(), kv_len.data_ptr(), work.data_ptr(), split.data_ptr(), n_work,
            _ptr(combine), n_combine, out.data_ptr(), out.stride(0), q_heads, kv_heads, head_dim,
            block_size, ws.data_ptr(), need, _stream())
    _lib.check(rc, "sp_attention_prefill_split")


def a2a_pack(src: torch.Tensor, dst: torch.Tensor, rows: int, peers: int, width: int) -> None:
    if rows == 0:
        return
    _lib.check(_lib.load().sp_a2a_pack(src.data_ptr(), src.stride(0), dst.data_ptr(), rows, peers,
                                       width, _stream()), "sp_a2a_pack")


def a2a_unpack(src: torch.Tensor, dst: torch.Tensor, rows: int, peers: int, width: int) -> None:
    if rows == 0:
        return
    _lib.check(_lib.load().sp_a2a_unpack(src.data_ptr(), dst.data_ptr(), dst.stride(0), rows,
                                         peers, width, _stream()), "sp_a2a_unpack")


def add_f32(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor) -> None:
    _need(a, torch.float32, "add a")
    n = a.numel()
    if n == 0:
        return
    _lib.check(_lib.load().sp_add_f32(a.data_ptr(), b.data_ptr(), out.data_ptr(), n, _stream()),
               "sp_add_f32")


def add_f64(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor) -> None:
    _need(a, torch.float64, "add a")
    _need(b, torch.float64, "add b")
    _need(out, torch.float64, "add out")
    if a.numel():
        _lib.check(_lib.load().sp_add_f64(a.data_ptr(), b.data_ptr(), out.data_ptr(), a.numel(),
                                          _stream()), "sp_add_f64")


def argmax(logits: torch.Tensor, idx: torch.Tensor, val: Optional[torch.Tensor] = None) -> None:
    _need(logits, torch.float32, "argmax logits")
    rows, vocab = logits.shape
    if rows == 0:
        return
    _lib.check(_lib.load().sp_argmax(logits.data_ptr(), logits.stride(0), rows, vocab,
                                     idx.data_ptr(), _ptr(val), _stream()), "sp_argmax")


def gather_rows(src: torch.Tensor, idx: torch.Tensor, dst: torch.Tensor) -> None:
    rows = idx.shape[0]
    if rows == 0:
        return
    _lib.check(_lib.load().sp_gather_rows_f32(src.data_ptr(), src.stride(0), idx.data_ptr(),
                                              dst.data_ptr(), dst.stride(0), rows, src.shape[1],
                                              _stream()), "sp_gather_rows_f32")


def rms_norm_f32(x: torch.Tensor, gain: torch.Tensor, eps: float, out: torch.Tensor) -> None:
    """out = gain * x / sqrt(mean(x^2) + eps) per row, f32 (sp_rms_norm_f32)."""
    _need(x, torch.float32, "rms_norm x")
    _need(gain, torch.float32, "rms_norm gain")
    _need(out, torch.float32, "rms_norm out")
    rows, hidden = x.shape
    _lib.check(_lib.load().sp_rms_norm_f32(x.data_ptr(), x.stride(0), gain.data_ptr(), float(eps),
                                           out.data_ptr(), out.stride(0), rows, hidden, _stream()),
               "sp_rms_norm_f32")


def gelu_f32(x: torch.Tensor, out: torch.Tensor) -> None:
    """tanh-form GeLU, elementwise f32 (sp_gelu_f32); x and out contiguous."""
    _need(x, torch.float32, "gelu x")
    _need(out, torch.float32, "gelu out")
    _lib.check(_lib.load().sp_gelu_f32(x.data_ptr(), out.data_ptr(), x.numel(), _stream()),
               "sp_gelu_f32")


def softmax_rows_f32(x: torch.Tensor, out: torch.Tensor) -> None:
    """Row softmax with shift-by-max, f32 (sp_softmax_rows_f32)."""
    _need(x, torch.float32, "softmax x")
    _need(out, torch.float32, "softmax out")
    rows, width = x.shape
    _lib.check(_lib.load().sp_softmax_rows_f32(x.data_ptr(), x.stride(0), out.data_ptr(),
                                               out.stride(0), rows, width, _stream()),
               "sp_softmax_rows_f32")

