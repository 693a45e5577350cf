"""CPU-only tests of the product's host side: the C-ABI library loads and
exports every symbol include/shiftpar.h declares, and the integer/host logic
(paged allocator, shard bounds, policy, weight layouts, FLOP mirror, KV cache
bookkeeping) matches the oracle / reference semantics bit-exactly."""

import os
import re

import numpy as np
import pytest
import torch

import oracle
from oracle.kvcache import PagedAllocator
from oracle.model import init_weights_llama, llama_tiny_config
from oracle.prims import rope_tables, sinusoidal_positions

from helpers import host_dict, product_config

from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, ConfigError, ContractViolation,
                                   ParallelMode, PassShape, ShiftPolicy, SwiftKvConfig, choose_mode,
                                   default_token_threshold, flop_count, partition_heads,
                                   shard_bounds, shard_rows)
from paper_2507_11830_b200 import _lib
from paper_2507_11830_b200.config import llama31_8b, llama33_70b, tiny_llama
from paper_2507_11830_b200.kv_cache import BlockAllocator, KvCache, KvPool
from paper_2507_11830_b200.weights import ModelWeights, rope_table, sinusoidal_table

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    src = open(os.path.join(ROOT, "include", "shiftpar.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(sp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import ctypes
    if not os.path.exists(_lib.LIB_PATH):
        from paper_2507_11830_b200 import build
        build.build()
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 14
    for s in syms:
        assert hasattr(lib, s), s
    assert sorted(_lib.SIGNATURES) == syms
    loaded = _lib.load()
    assert loaded.sp_abi_version() == 1


def test_library_missing_fails_loudly(monkeypatch, tmp_path):
    from paper_2507_11830_b200.errors import LibraryMissing
    monkeypatch.setattr(_lib, "_lib", None)
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "nope.so"))
    with pytest.raises(LibraryMissing):
        _lib.load()


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_2507_11830_b200")
    for f in os.listdir(pkg):
        if f.endswith(".py"):
            src = open(os.path.join(pkg, f)).read()
            assert not re.search(r"^\s*(from|import)\s+oracle", src, re.M), f


def test_allocator_matches_oracle_bitexact():
    rng = np.random.default_rng(0)
    a, b = BlockAllocator(64, 16), PagedAllocator(64, 16)
    lens = {}
    for step in range(300):
        key = int(rng.integers(0, 8))
        if rng.random() < 0.15 and key in lens:
            a.release(key)
            b.release(key)
            lens.pop(key)
            continue
        n = lens.get(key, 0) + int(rng.integers(1, 40))
        if a.blocks_needed(key, n) > a.free_blocks:
            assert b.blocks_needed(key, n) > b.free_blocks
            continue
        a.reserve(key, n)
        b.reserve(key, n)
        start = lens.get(key, 0)
        lens[key] = n
        np.testing.assert_array_equal(a.slots(key, start, n - start),
                                      b.slots(key, np.arange(start, n)))
        assert a.tables[key] == b.tables[key]
    assert a.free_blocks == b.free_blocks


def test_shard_bounds_and_partition(golden):
    _, meta = golden
    assert shard_rows(10, 4) == meta["shard_rows"]["10_4"] == oracle.shard_rows(10, 4)
    assert shard_rows(1, 2) == [1, 0]
    for m in range(0, 40):
        for p in (1, 2, 3, 4, 8):
            assert shard_bounds(m, p) == oracle.shard_bounds(m, p)
    assert [list(x) for x in partition_heads(8, 4)] == meta["partition_heads_8_4"]
    with pytest.raises(ConfigError):
        partition_heads(6, 4)


class _Seq:
    def __init__(self):
        self.cache = object()


def test_policy_and_batch_validation():
    s = [_Seq() for _ in range(4)]
    small = Batch(BatchKind.DECODE, [BatchItem(s[0], [1])])
    at = Batch(BatchKind.DECODE, [BatchItem(x, [1]) for x in s])
    pol = ShiftPolicy(token_threshold=4)
    assert choose_mode(pol, small) is ParallelMode.TP
    assert choose_mode(pol, at) is ParallelMode.SP
    assert choose_mode(ShiftPolicy.fixed_sp(), small) is ParallelMode.SP
    assert choose_mode(ShiftPolicy.fixed_tp(), at) is ParallelMode.TP
    assert default_token_threshold(8) == 32
    with pytest.raises(ConfigError):
        ShiftPolicy(token_threshold=0).validate()
    with pytest.raises(ConfigError):
        ShiftPolicy(kind="shift").validate()
    with pytest.raises(ContractViolation):
        Batch(BatchKind.PREFILL, []).validate()
    with pytest.raises(ContractViolation):
        Batch(BatchKind.PREFILL, [BatchItem(s[0], [])]).validate()
    with pytest.raises(ContractViolation):
        Batch(BatchKind.DECODE, [BatchItem(s[0], [1, 2])]).validate()
    Batch(BatchKind.DECODE, [BatchItem(s[0], [1, 2])], speculative=True).validate()
    with pytest.raises(ContractViolation):
        Batch(BatchKind.DECODE, [BatchItem(s[0], [1]), BatchItem(s[0], [2])]).validate()
    assert SwiftKvConfig(True).resolve_cut(4) == 2
    assert SwiftKvConfig(False).resolve_cut(4) == 4
    with pytest.raises(ConfigError):
        SwiftKvConfig(True, 0).resolve_cut(4)


@pytest.mark.parametrize("mode", ["tp", "sp"])
@pytest.mark.parametrize("p", [1, 2, 4, 8])
def test_flop_mirror_matches_oracle(mode, p):
    ocfg = llama_tiny_config(n_heads=8, n_kv_heads=8 if p == 8 else 4)
    cfg = product_config(ocfg)
    for spans, hist, span_logits, cut in [((9, 5), (0, 0), False, None), ((1, 1, 1), (9, 5, 3), False, None),
                                          ((7, 3), (2, 0), True, None), ((20, 11, 3), (0, 0, 0), False, 2)]:
        got = flop_count(PassShape(spans, hist, span_logits), mode, cfg, p, swiftkv_cut=cut)
        want = oracle.flop_count(spans, hist, mode, ocfg, p, span_logits=span_logits, swiftkv_cut=cut)
        assert got == want


def test_rope_and_position_tables_match_oracle_bitexact():
    from paper_2507_11830_b200.config import LLAMA3_ROPE_SCALING
    a = rope_table(4096, 128, 500000.0, LLAMA3_ROPE_SCALING)
    b = rope_tables(4096, 128, 500000.0, LLAMA3_ROPE_SCALING)
    assert a.tobytes() == b.tobytes()
    assert sinusoidal_table(64, 256).tobytes() == sinusoidal_positions(np.arange(64), 256,
                                                                       dtype=np.float32).tobytes()


@pytest.mark.parametrize("p", [1, 2, 4])
def test_weight_layouts_are_zero_copy_tp_views(p):
    """Fused/permuted replica: rank r's q|k|v rows, interleaved gate/up rows and
    K windows are exactly the reference TP shards (model.py:220-281)."""
    ocfg = llama_tiny_config(n_kv_heads=4, n_layers=1)
    ow = init_weights_llama(ocfg, seed=3)
    w = ModelWeights.from_host(product_config(ocfg), host_dict(ow), p, device="cpu")
    lw, olw = w.layers[0], ow.layers[0]
    d, hq, hk = ocfg.head_dim, ocfg.n_heads // p, ocfg.kv_heads // p
    W = w.qkv_width
    f = ocfg.ffn_dim // p

    def bf(x):
        return torch.as_tensor(np.ascontiguousarray(x.T)).to(torch.bfloat16)

    for r in range(p):
        blk = lw.wqkv[r * W:(r + 1) * W]
        assert blk.data_ptr() == lw.wqkv.data_ptr() + r * W * ocfg.hidden * 2
        assert torch.equal(blk[:hq * d], bf(olw["wq"][:, r * hq * d:(r + 1) * hq * d]))
        assert torch.equal(blk[hq * d:(hq + hk) * d], bf(olw["wk"][:, r * hk * d:(r + 1) * hk * d]))
        assert torch.equal(blk[(hq + hk) * d:], bf(olw["wv"][:, r * hk * d:(r + 1) * hk * d]))
        gu = lw.wgu[r * 2 * f:(r + 1) * 2 * f].view(f // 128, 2, 128, -1)
        assert torch.equal(gu[:, 0].reshape(f, -1), bf(olw["w_gate"][:, r * f:(r + 1) * f]))
        assert torch.equal(gu[:, 1].reshape(f, -1), bf(olw["w_up"][:, r * f:(r + 1) * f]))
        assert torch.equal(lw.wdown[:, r * f:(r + 1) * f], bf(olw["w_down"][r * f:(r + 1) * f, :]))
        assert torch.equal(lw.wo[:, r * hq * d:(r + 1) * hq * d], bf(olw["wo"][r * hq * d:(r + 1) * hq * d, :]))


def test_kvcache_bookkeeping_semantics():
    """Staged vs committed, per-layer cursors, overflow, logical truncate,
    write counter, fingerprint (reference tests/test_kv_cache.py)."""
    pool = KvPool(2, ((0, 2), (2, 4)), 8, 16, 4, [0, 1], torch.device("cpu"))
    c = KvCache(pool, 0, 8)
    c._stage(0, 0, 3)
    with pytest.raises(ContractViolation):
        c.commit(3)
    for dev, layer in ((0, 1), (1, 0), (1, 1)):
        c._stage(dev, layer, 3)
    assert c.token_count == 0
    c.commit(3)
    assert c.token_count == 3
    assert c.device_write_counter(0) == 2 * 3 * 2 * 8 * 2 * 2  # layers*tokens*heads*dim*bf16*(K,V)
    before = c.write_counter
    c.truncate(1)
    assert c.token_count == 1 and c.write_counter == before
    with pytest.raises(ContractViolation):
        c.truncate(2)
    from paper_2507_11830_b200.errors import CacheOverflow
    with pytest.raises(CacheOverflow):
        c._stage(0, 0, 9)
    fp = c.fingerprint()
    assert fp.axis_order == "layer,head,token,dim" and fp.heads_per_device == 2
    assert fp.world_size == 2 and fp.precision == "bf16"


def test_presets_validate():
    for cfg, worlds in ((tiny_llama(), (1, 2)), (llama31_8b(), (1, 2, 4, 8)),
                        (llama33_70b(), (1, 2, 4, 8))):
        cfg.validate()
        for p in worlds:
            cfg.check_world(p)
    with pytest.raises(ConfigError):
        tiny_llama().check_world(4)  # 2 kv heads cannot split 4 ways
    assert llama31_8b().hidden == 4096 and llama33_70b().n_layers == 80


def test_attention_split_plan_covers_every_key_tile_once():
    """Split-KV plan (SP=8 shape: one 8K request, 4 q / 1 kv head per rank):
    every work tile's key tiles are covered exactly once by its entries, split
    tiles own contiguous slots listed in their combine entry, no piece exceeds
    the chunk, entries are longest first; enough tiles -> no plan."""
    from paper_2507_11830_b200.engine import attention_split_plan
    T, tt = 8192, 64
    wl = sorted([(0, t0, t0) for t0 in range(0, T, tt)], key=lambda w: -w[2])
    plan = attention_split_plan(wl, [T], [0], tt, hk=1, sms=148, max_slots=4096)
    assert plan is not None
    work, split, comb, n_slots = plan
    sizes = split[:, 1] - split[:, 0]
    assert (sizes > 0).all() and list(sizes) == sorted(sizes, reverse=True)
    total = sum(-(-(t0 + tt) // 128) for _, t0, _ in wl)
    assert sizes.max() <= max(2, -(-total // 148))
    cover = {}
    for (i, t0), (jb, je, slot, _) in zip(work.tolist(), split.tolist()):
        cover.setdefault((i, t0), []).append((jb, je, slot))
    slots_seen = []
    for (i, t0), parts in cover.items():
        parts.sort()
        n_kt = -(-(t0 + tt) // 128)
        assert parts[0][0] == 0 and parts[-1][1] == n_kt
        assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
        if len(parts) == 1:
            assert parts[0][2] == -1
        else:
            c = [x for x in comb.tolist() if (x[0], x[1]) == (i, t0)]
            assert len(c) == 1 and c[0][3] == len(parts)
            assert [p[2] for p in parts] == list(range(c[0][2], c[0][2] + len(parts)))
            slots_seen += [p[2] for p in parts]
    assert sorted(slots_seen) == list(range(n_slots))
    # a pass that already fills the GPU, or a workspace too small: no plan
    assert attention_split_plan(wl, [T], [0], tt, hk=8, sms=148, max_slots=4096) is None
    assert attention_split_plan(wl, [T], [0], tt, hk=1, sms=148, max_slots=1) is None


@pytest.mark.parametrize("M,N,epi,want", [
    (1, 4096, 1, 0), (64, 4096, 5, 0), (256, 4096, 2, 0),    # decode: swap-AB (M <= 256)
    (1024, 4096, 2, 1), (8192, 6144, 0, 1),                   # prefill: 2-CTA pairs
    (512, 4096, 2, 128), (512, 6144, 0, 1),                   # wave model at small per-rank M
    (300, 28672, 3, 1), (1, 128256, 1, 0),                    # SwiGLU forces 256; LM head row: swap-AB
    (32, 57344, 3, 0), (64, 128256, 1, 256),                  # >= 1 weight tile per SM: swap-AB to 32 rows
    (64, 28672, 3, 0), (128, 28672, 3, 256), (256, 6144, 1, 0)])  # wide N leaves swap-AB above 64 rows
def test_gemm_plan_regimes(M, N, epi, want, monkeypatch):
    """The host-side GEMM plan (sp_gemm_plan, the one function sp_gemm_bf16
    dispatches on) picks the documented regime per shape on 148 SMs."""
    import ctypes
    lib = _lib.load()
    for k in ("SP_GEMM_NO_SPLITK", "SP_GEMM_FORCE_BN", "SP_GEMM_2CTA"):
        monkeypatch.delenv(k, raising=False)
    # a registered split-K workspace (address only: planning never touches it)
    assert lib.sp_gemm_set_workspace(ctypes.c_void_p(1 << 24), 64 << 20) == 0
    try:
        assert lib.sp_gemm_plan(M, N, 4096, epi, 148) == want
        monkeypatch.setenv("SP_GEMM_NO_SPLITK", "1")  # tests pin the non-decode regime this way
        assert lib.sp_gemm_plan(M, N, 4096, epi, 148) != 0
    finally:
        lib.sp_gemm_set_workspace(None, 0)


def test_gemm_plan_follows_dispatch_overrides(monkeypatch):
    """the plan reports what the dispatcher runs — no workspace
    means no K-split swap-AB (raw partials need none), and FORCE_BN=256 with
    SP_GEMM_2CTA=0 is a 1-CTA 128x256 tile, not a pair."""
    lib = _lib.load()
    for k in ("SP_GEMM_NO_SPLITK", "SP_GEMM_FORCE_BN", "SP_GEMM_2CTA"):
        monkeypatch.delenv(k, raising=False)
    lib.sp_gemm_set_workspace(None, 0)
    assert lib.sp_gemm_partials(1, 4096, 4096) > 1
    assert lib.sp_gemm_plan(1, 4096, 4096, 1, 148) != 0     # split-K swap needs the workspace
    assert lib.sp_gemm_plan(1, 4096, 4096, 5, 148) == 0     # partial epilogue writes into D
    monkeypatch.setenv("SP_GEMM_FORCE_BN", "256")
    monkeypatch.setenv("SP_GEMM_2CTA", "0")
    assert lib.sp_gemm_plan(8192, 6144, 4096, 0, 148) == 256
    monkeypatch.delenv("SP_GEMM_2CTA")
    assert lib.sp_gemm_plan(8192, 6144, 4096, 0, 148) == 1


def test_b200_crossover_model():
    """default_token_threshold with a geometry = the B200 cost-model crossover
    (shift_cost): TP wins decode-size passes, SP wins every pass from tau up,
    tau sits between the reference's 4P and one 8K prefill, and 4P stays the
    geometry-free default.  (tau is not monotone in P: the GEMM regime and the
    one-/two-shot all-reduce switch at fixed row counts.)"""
    from paper_2507_11830_b200 import llama31_8b, llama33_70b
    from paper_2507_11830_b200.shift_cost import comm_us, crossover, pass_us
    for cfg in (llama31_8b(), llama33_70b()):
        taus = [default_token_threshold(p, cfg) for p in (2, 4, 8)]
        assert all(4 * p < t <= 8192 for p, t in zip((2, 4, 8), taus))
        assert default_token_threshold(1, cfg) == 1
        for p, tau in zip((2, 4, 8), taus):
            assert tau == crossover(cfg, p)
            for m in (1, 8, 64):
                assert pass_us(cfg, "tp", p, m) < pass_us(cfg, "sp", p, m)
            for m in (tau, 2 * tau, 8192, 32768):
                assert pass_us(cfg, "sp", p, m) <= pass_us(cfg, "tp", p, m)
            # SP moves ~P x fewer collective bytes than TP at prefill sizes
            assert comm_us(cfg, "sp", p, 8192) < comm_us(cfg, "tp", p, 8192)
    assert default_token_threshold(8) == 32
    with pytest.raises(ConfigError):
        default_token_threshold(0)


def test_decode_layer_args_layout_matches_header(tmp_path):
    """The ctypes mirror of sp_decode_layer_args / sp_dl_proj has the C layout
    (offsets and sizes from gcc on include/shiftpar.h)."""
    import ctypes
    import shutil
    import subprocess
    if shutil.which("gcc") is None:
        pytest.skip("no gcc")
    fields = [f for f, _ in _lib.DecodeLayerArgs._fields_]
    pfields = [f for f, _ in _lib.DlProj._fields_]
    src = tmp_path / "lay.c"
    src.write_text(
        '#include <stdio.h>\n#include <stddef.h>\n#include "shiftpar.h"\nint main(void){\n'
        'printf("%zu\\n", sizeof(sp_decode_layer_args));\n'
        'printf("%zu\\n", sizeof(sp_dl_proj));\n'
        + "".join(f'printf("%zu\\n", offsetof(sp_decode_layer_args, {f}));\n' for f in fields)
        + "".join(f'printf("%zu\\n", offsetof(sp_dl_proj, {f}));\n' for f in pfields)
        + "return 0;}\n")
    exe = tmp_path / "lay"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), str(src), "-o", str(exe)],
                   check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True,
                                          check=True).stdout.split()]
    want = [ctypes.sizeof(_lib.DecodeLayerArgs), ctypes.sizeof(_lib.DlProj)]
    want += [getattr(_lib.DecodeLayerArgs, f).offset for f in fields]
    want += [getattr(_lib.DlProj, f).offset for f in pfields]
    assert got == want
