"""ctypes binding of libshiftpar.so — the C-ABI declared in include/shiftpar.h.

The library is built in-tree (``python -m paper_2507_11830_b200.build`` or
``__graft_entry__.build()``) and loaded from the package directory.  There is
no fallback: if the library is missing every op raises ``LibraryMissing``.
"""

from __future__ import annotations

import ctypes
import os

from .errors import ContractViolation, LibraryMissing

LIB_NAME = "libshiftpar.so"
LIB_PATH = os.environ.get("SP_LIB_PATH") or os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME)  # override: A/B kernel comparisons

_c_int = ctypes.c_int
_i64 = ctypes.c_int64
_vp = ctypes.c_void_p
_f32 = ctypes.c_float

# name -> (restype, argtypes); must match include/shiftpar.h exactly
SIGNATURES = {
    "sp_last_error": (ctypes.c_char_p, []),
    "sp_abi_version": (_c_int, []),
    "sp_kernel_launches": (_i64, []),
    "sp_device_check": (_c_int, [ctypes.POINTER(_c_int)]),
    "sp_step_trace_bind": (_c_int, [_vp, _vp, _c_int]),
    "sp_gemm_bf16": (_c_int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _i64, _c_int, _c_int, _c_int,
                              _c_int, _i64, _i64, _vp]),
    "sp_gemm_set_workspace": (_c_int, [_vp, _i64]),
    "sp_gemm_bf16_to_peers": (_c_int, [_vp, _i64, _i64, _i64, _vp, _i64, _vp, _vp, _i64, _i64,
                                       _c_int, _c_int, _c_int, _c_int, _i64, _vp]),
    "sp_peer_scatter_rows": (_c_int, [_vp, _i64, _c_int, _c_int, _c_int, _c_int, _vp, _vp]),
    "sp_peer_signal": (_c_int, [_vp, _c_int, _c_int, _vp]),
    "sp_peer_wait": (_c_int, [_vp, _c_int, _vp]),
    "sp_peer_allreduce_add_rmsnorm": (_c_int, [_vp, _c_int, _c_int, _vp, _i64, _vp, _f32, _vp, _i64,
                                               _c_int,
                                               _c_int, _vp]),
    "sp_peer_reduce_scatter_rmsnorm": (_c_int, [_vp, _c_int, _c_int, _vp, _i64, _vp, _f32, _vp,
                                                _i64, _c_int, _c_int, _vp]),
    "sp_embed": (_c_int, [_vp, _vp, _vp, _vp, _vp, _c_int, _c_int, _vp]),
    "sp_add_rmsnorm": (_c_int, [_vp, _i64, _vp, _c_int, _vp, _f32, _vp, _vp, _i64, _c_int, _c_int,
                                _vp]),
    "sp_gemm_partials": (_c_int, [_c_int, _c_int, _c_int]),
    "sp_gemm_plan": (_c_int, [_c_int, _c_int, _c_int, _c_int, _c_int]),
    "sp_ipc_export": (_c_int, [_vp, _vp, ctypes.POINTER(_i64)]),
    "sp_attention_prefill_split": (_c_int, [_vp, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp,
                                            _vp, _vp, _vp, _c_int, _vp, _c_int, _vp, _i64, _c_int,
                                            _c_int, _c_int, _c_int, _vp, _i64, _vp]),
    "sp_ipc_import": (_c_int, [_vp, _i64, ctypes.POINTER(_vp)]),
    "sp_rope_kv_write_partials": (_c_int, [_vp, _c_int, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp,
                                           _c_int, _c_int, _c_int, _c_int, _c_int, _vp]),
    "sp_rope_kv_write": (_c_int, [_vp, _i64, _vp, _vp, _vp, _vp, _i64, _vp, _vp, _c_int, _c_int,
                                  _c_int, _c_int, _c_int, _vp]),
    "sp_gemm_bf16_qkv_rope": (_c_int, [_vp, _i64, _vp, _i64, _c_int, _c_int, _vp, _vp, _vp, _vp,
                                       _i64, _vp, _vp, _c_int, _c_int, _c_int, _vp]),
    "sp_attention": (_c_int, [_vp, _i64, _i64, _vp, _vp, _i64, _vp, _i64, _vp, _vp, _vp, _c_int,
                              _vp, _c_int, _c_int, _c_int, _vp, _i64, _c_int, _c_int, _c_int,
                              _c_int, _vp, _i64, _vp]),
    "sp_attn_workspace_bytes": (_i64, [_c_int, _c_int, _c_int, _c_int]),
    "sp_attention_decode_qkv": (_c_int, [_vp, _c_int, _i64, _c_int, _vp, _vp, _vp, _vp, _vp, _i64,
                                         _vp, _i64, _vp, _vp, _c_int, _c_int, _vp, _i64, _c_int,
                                         _c_int, _c_int, _vp, _i64, _vp]),
    "sp_attn_tile_tokens": (_c_int, [_c_int, _c_int, _c_int, _c_int]),
    "sp_a2a_pack": (_c_int, [_vp, _i64, _vp, _c_int, _c_int, _c_int, _vp]),
    "sp_a2a_unpack": (_c_int, [_vp, _vp, _i64, _c_int, _c_int, _c_int, _vp]),
    "sp_add_f32": (_c_int, [_vp, _vp, _vp, _i64, _vp]),
    "sp_argmax": (_c_int, [_vp, _i64, _c_int, _c_int, _vp, _vp, _vp]),
    "sp_gather_rows_f32": (_c_int, [_vp, _i64, _vp, _vp, _i64, _c_int, _c_int, _vp]),
    "sp_gather_rows_bf16": (_c_int, [_vp, _i64, _vp, _vp, _i64, _c_int, _c_int, _vp]),
    "sp_rms_norm_f32": (_c_int, [_vp, _i64, _vp, _f32, _vp, _i64, _c_int, _c_int, _vp]),
    "sp_gelu_f32": (_c_int, [_vp, _vp, _i64, _vp]),
    "sp_add_f64": (_c_int, [_vp, _vp, _vp, _i64, _vp]),
    "sp_softmax_rows_f32": (_c_int, [_vp, _i64, _vp, _i64, _c_int, _c_int, _vp]),
}



class DlProj(ctypes.Structure):
    """sp_dl_proj (include/shiftpar.h)."""
    _fields_ = [("w", _vp), ("ldw", _i64), ("x", _vp), ("ldx", _i64), ("n", _c_int),
                ("k", _c_int), ("kind", _c_int), ("pad_", _c_int), ("gain", _vp), ("out", _vp),
                ("ldo", _i64)]


class DecodeLayerArgs(ctypes.Structure):
    """sp_decode_layer_args (include/shiftpar.h)."""
    _fields_ = [("rows", _c_int), ("hidden", _c_int), ("x", _vp), ("ldx", _i64), ("eps", _f32),
                ("n_proj", _c_int), ("proj", DlProj * 4), ("lead_gain", _vp), ("lead_out", _vp),
                ("ld_lead", _i64), ("pos", _vp), ("slot", _vp), ("rope", _vp), ("q_out", _vp),
                ("ldq", _i64), ("k_pool", _vp), ("v_pool", _vp), ("q_heads", _c_int),
                ("kv_heads", _c_int), ("block_size", _c_int), ("head_dim", _c_int), ("ws", _vp),
                ("ws_bytes", _i64), ("sync", _vp)]


SIGNATURES["sp_decode_layer"] = (_c_int, [ctypes.POINTER(DecodeLayerArgs), _vp])
SIGNATURES["sp_decode_layer_ws_bytes"] = (_i64, [ctypes.POINTER(DecodeLayerArgs)])

_lib = None


def load():
    """Load libshiftpar.so (once).  Raises LibraryMissing if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} not found: build it with `python -m paper_2507_11830_b200.build` "
            "(there is no CPU fallback)")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def exported_symbols():
    return sorted(SIGNATURES)


def check(rc: int, what: str) -> None:
    if rc != 0:
        msg = load().sp_last_error().decode(errors="replace")
        raise ContractViolation(f"{what} failed (status {rc}): {msg}")
