"""Parity at the BASELINE shapes (VERDICT r1 "Next" #1).

The bench workload's dominant kernels — the 2-CTA pair GEMM, the fused
QKV-RoPE epilogue, full-length tcgen05 attention, the swap-AB decode GEMMs and
the SwiftKV tails — checked numerically at the sizes the bench runs them,
against ``tests/torch_ref.py`` (a torch fp32 restatement of the oracle forward,
TF32 off, pinned to the numpy oracle by ``tests/test_torch_ref.py``):

* Llama-3.1-8B geometry, 32 layers, one 8192-token SP prefill (the bench
  step): last-row logits through the bench's call, sampled rows through
  ``span_logits``, and K/V of sampled layers;
* B=64 requests at ctx 2K, three teacher-forced TP decode steps (eager,
  capture, graph replay): logits of every request, slot mappings and block
  tables bit-exact vs the oracle's integer allocator;
* SwiftKV 32K-token prefill at cut 16;
* P=8 loopback (one kv head per rank, 8B widths) SP and TP: logits and K/V vs
  the same fp32 forward, slot mappings vs the oracle's integer allocator.

Tolerance (north star "within a stated bf16 tolerance", e.g. 2e-2): max |got -
want| / max |want| <= 2e-2 for logits and K/V wherever bf16 storage itself
stays under that — the 8192-token prefill at 2 layers, the P=8 tests.  At the
full 32-layer depth of this random-init model the bf16 storage points alone
move the fp32 result by 4-6% (measured: the SAME fp32 forward with bf16
rounding at the GPU's storage points — activations, q/k/v, attention output,
SwiGLU product and the attention probabilities P (``emulate_bf16`` +
``round_p``) — differs from plain fp32 by ~0.05 at 8K; fp32 vs f64 differs by
3e-5, so this is rounding amplified through 32 layers, not arithmetic —
tools/parity_depth.py, profiles/r02_parity_depth.json).  There the bar is:
error vs fp32 <= max(2e-2, 1.25 x that bf16 floor), the floor computed in
the same test on the same rows, and the product closer to the bf16-emulated
forward than plain fp32 is.
Integers exact.  Set SP_PARITY_LOG=<file> to append the measured errors.
"""

import json
import os

import numpy as np
import pytest
import torch

from oracle.kvcache import PagedAllocator
from oracle.model import init_weights_llama, llama_tiny_config

import torch_ref
from helpers import device_weights, rel_err

pytestmark = pytest.mark.gpu

LOGIT_TOL = 2e-2
KV_TOL = 2e-2
BF16_FLOOR_FACTOR = 1.25   # full-depth bar: <= 1.25 x the bf16-emulated forward's own error


def _depth_tol(floor: float) -> float:
    return max(LOGIT_TOL, BF16_FLOOR_FACTOR * floor)

from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, SwiftKvConfig, llama31_8b)
from paper_2507_11830_b200.weights import ModelWeights  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


def _log(name, **vals):
    path = os.environ.get("SP_PARITY_LOG")
    print(name, vals)
    if path:
        with open(path, "a") as f:
            f.write(json.dumps({"test": name, **vals}) + "\n")


def _tokens(seed, n, vocab):
    return [int(t) for t in np.random.default_rng(seed).integers(0, vocab, size=n)]


@pytest.fixture(scope="module")
def w8b():
    """The bench's weights: 8B geometry, 32 layers, seed 0, drawn on the device."""
    cfg = llama31_8b(max_seq=32768)
    w = ModelWeights.random(cfg, seed=0, world_size=1)
    yield w
    del w
    torch.cuda.empty_cache()


@pytest.fixture(scope="module")
def rw8b(w8b):
    """fp32 copies of the 32 layers (~28 GB), made once for all forwards."""
    rw = torch_ref.RefWeights.from_model(w8b).keep_layers()
    yield rw
    del rw
    torch.cuda.empty_cache()


def _prefill_8k(w, rw, n, emulate_floor: bool):
    prompt = _tokens(0, n, w.config.vocab_size)
    eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_sp(), num_blocks=2 * n // 64 + 8)
    a = eng.new_sequence(0, capacity=n)
    last, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(a, prompt)]), mode=ParallelMode.SP)
    b = eng.new_sequence(1, capacity=n)
    span, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(b, prompt)]), mode=ParallelMode.SP,
                       span_logits=True)
    rows = [0, 1, 63, 64, 1000, 2047, 4095, 6000, n - 1]
    want, cache = torch_ref.forward(rw, prompt, logit_rows=rows)
    res = {"last": rel_err(last[0].cpu().numpy(), want[-1].cpu().numpy()),
           "span": rel_err(span[0][rows].cpu().numpy(), want.cpu().numpy())}
    kv = {}
    L = w.config.n_layers
    for layer in sorted({0, L // 2, L - 1}):
        for head in (0, 7):
            kg, vg = a.cache.read_window(0, layer, head)
            kw, vw = cache.k[layer][:, head], cache.v[layer][:, head]
            kv[f"L{layer}h{head}"] = max(rel_err(kg.float().cpu().numpy(), kw.cpu().numpy()),
                                         rel_err(vg.float().cpu().numpy(), vw.cpu().numpy()))
            kb, vb = b.cache.read_window(0, layer, head)
            assert torch.equal(kg, kb) and torch.equal(vg, vb)   # same pass, same bits
    res["kv_max"] = max(kv.values())
    if emulate_floor:
        emu, ecache = torch_ref.forward(rw, prompt, logit_rows=rows, emulate_bf16=True,
                                        round_p=True)
        res["floor_span"] = rel_err(emu.cpu().numpy(), want.cpu().numpy())
        res["floor_last"] = rel_err(emu[-1].cpu().numpy(), want[-1].cpu().numpy())
        res["floor_kv"] = max(rel_err(ecache.k[l][:, 0].cpu().numpy(), cache.k[l][:, 0].cpu().numpy())
                              for l in range(L))
        res["vs_emulated"] = rel_err(span[0][rows].cpu().numpy(), emu.cpu().numpy())
    s_ = np.sort(want[-1].cpu().numpy())
    res["greedy_decisive"] = bool(s_[-1] - s_[-2] > 2 * res["last"] * np.abs(s_).max())
    res["greedy_equal"] = int(torch.argmax(last[0])) == int(torch.argmax(want[-1]))
    return res


def test_8b_width_8k_prefill_2layers():
    """8192 tokens at 8B widths (pair GEMM at M=8192, fused QKV-RoPE, full
    causal tcgen05 attention) at a depth where 2e-2 is the bar."""
    cfg = llama31_8b(n_layers=2, max_seq=8192)
    w = ModelWeights.random(cfg, seed=0, world_size=1)
    res = _prefill_8k(w, torch_ref.RefWeights.from_model(w), 8192, emulate_floor=False)
    _log("8b_2l_8k_sp_prefill", **res)
    assert res["last"] <= LOGIT_TOL and res["span"] <= LOGIT_TOL
    assert res["kv_max"] <= KV_TOL
    if res["greedy_decisive"]:
        assert res["greedy_equal"]


def test_8b_32layer_8k_sp_prefill(w8b, rw8b):
    """The bench step itself (32 layers, 8192 tokens, SP)."""
    res = _prefill_8k(w8b, rw8b, 8192, emulate_floor=True)
    _log("8b_32l_8k_sp_prefill", **res)
    # like for like: the returned row against the bf16 floor of that row, the
    # sampled rows against the floor over the same rows
    assert res["last"] <= _depth_tol(res["floor_last"])
    assert res["span"] <= _depth_tol(res["floor_span"])
    assert res["kv_max"] <= max(KV_TOL, BF16_FLOOR_FACTOR * res["floor_kv"])
    # the product follows the bf16 trajectory: closer to it than plain fp32 is
    assert res["vs_emulated"] < res["floor_span"]
    if res["greedy_decisive"]:
        assert res["greedy_equal"]


def test_8b_b64_ctx2k_decode(w8b, rw8b):
    B, ctx, steps = 64, 2048, 3
    vocab = w8b.config.vocab_size
    prompts = [_tokens(100 + i, ctx - steps, vocab) for i in range(B)]
    forced = [_tokens(200 + i, steps, vocab) for i in range(B)]
    eng = Engine(w8b, LoopbackGroup(1), ShiftPolicy.fixed_tp(), num_blocks=B * ctx // 64 + 8)
    oalloc = PagedAllocator(B * ctx // 64 + 8, 64)
    seqs = [eng.new_sequence(i, capacity=ctx) for i in range(B)]
    for lo in range(0, B, 8):  # 8 requests (16K tokens) per prefill pass
        items = [BatchItem(seqs[i], prompts[i]) for i in range(lo, lo + 8)]
        eng.step(Batch(BatchKind.PREFILL, items), mode=ParallelMode.SP)
        for i in range(lo, lo + 8):
            oalloc.reserve(i, len(prompts[i]))
    got = []
    for k in range(steps):
        lg, rec = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [forced[i][k]])
                                                    for i, s in enumerate(seqs)]),
                           mode=ParallelMode.TP)
        got.append(torch.stack(lg).cpu())
        t = len(prompts[0]) + k
        for i in range(B):
            oalloc.reserve(i, t + 1)
        want_slots = np.concatenate([oalloc.slots(i, [t]) for i in range(B)])
        assert np.array_equal(eng.last_slots, want_slots)
        bt = eng.last_block_table
        for i in range(B):
            tab = oalloc.tables[i]
            assert list(bt[i, :len(tab)]) == tab
    assert any(e.graph is not None for e in eng._graphs.values())  # step 3 replayed a graph
    rw = rw8b
    worst = floor = vs_emu = 0.0
    for i in range(B):
        _, cache = torch_ref.forward(rw, prompts[i], logit_rows=[])
        _, emu_cache = torch_ref.forward(rw, prompts[i], logit_rows=[], emulate_bf16=True,
                                         round_p=True)
        for k in range(steps):
            want, cache = torch_ref.forward(rw, [forced[i][k]], cache=cache)
            emu, emu_cache = torch_ref.forward(rw, [forced[i][k]], cache=emu_cache,
                                               emulate_bf16=True, round_p=True)
            w_, e_, g_ = want[0].cpu().numpy(), emu[0].cpu().numpy(), got[k][i].numpy()
            worst = max(worst, rel_err(g_, w_))
            floor = max(floor, rel_err(e_, w_))
            vs_emu = max(vs_emu, rel_err(g_, e_))
        del cache, emu_cache
    _log("8b_b64_ctx2k_tp_decode", worst=worst, floor=floor, vs_emulated=vs_emu)
    assert worst <= _depth_tol(floor)


def test_8b_swiftkv_32k_prefill(w8b, rw8b):
    n, cut = 32768, 16
    prompt = _tokens(1, n, w8b.config.vocab_size)
    eng = Engine(w8b, LoopbackGroup(1), ShiftPolicy.fixed_sp(),
                 swiftkv=SwiftKvConfig(enabled=True, cut_layer=cut), num_blocks=n // 64 + 8,
                 max_pass_tokens=n)
    s = eng.new_sequence(0, capacity=n)
    lg, rec = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]), mode=ParallelMode.SP)
    rw = rw8b
    want, cache = torch_ref.forward_swiftkv(rw, prompt, cut)
    emu, ecache = torch_ref.forward_swiftkv(rw, prompt, cut, emulate_bf16=True, round_p=True)
    floor = rel_err(emu[0].cpu().numpy(), want[0].cpu().numpy())
    kv_floor = max(rel_err(ecache.k[l][:, 3].cpu().numpy(), cache.k[l][:, 3].cpu().numpy())
                   for l in (cut - 1, cut, 31))
    del ecache
    err = rel_err(lg[0].cpu().numpy(), want[0].cpu().numpy())
    kv = []
    for layer in (cut - 1, cut, 31):
        kg, vg = s.cache.read_window(0, layer, 3)
        kv.append(rel_err(kg.float().cpu().numpy(), cache.k[layer][:, 3].cpu().numpy()))
        kv.append(rel_err(vg.float().cpu().numpy(), cache.v[layer][:, 3].cpu().numpy()))
    _log("8b_swiftkv_32k", logits=err, kv_max=max(kv), floor=floor, kv_floor=kv_floor)
    assert err <= _depth_tol(floor)
    assert max(kv) <= max(KV_TOL, BF16_FLOOR_FACTOR * kv_floor)


@pytest.fixture(scope="module")
def w8b_l2_host():
    cfg = llama_tiny_config(n_layers=2, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336,
                            vocab_size=128256, max_seq=1024)
    return init_weights_llama(cfg, seed=0)


@pytest.mark.parametrize("mode", [ParallelMode.SP, ParallelMode.TP])
def test_p8_loopback_8b_width(w8b_l2_host, mode):
    """P=8 (one kv head and four q heads per rank, 8B widths, 2 layers):
    uneven SP shards over two requests (span logits), then a decode step of
    one request (SP shards [1, 0, ..., 0]), against the fp32 dense forward on
    the same bf16 weights; slot mappings and block tables against the
    oracle's integer allocator."""
    P = 8
    ow = w8b_l2_host
    eng = Engine(device_weights(ow, P), LoopbackGroup(P), ShiftPolicy.fixed_tp())
    oalloc = PagedAllocator(eng.pool.num_blocks, eng.pool.block_size)
    rw = torch_ref.RefWeights.from_oracle(ow, device="cuda")
    prompts = [_tokens(11, 301, 128256), _tokens(12, 420, 128256)]
    seqs = [eng.new_sequence(i, capacity=768) for i in range(2)]
    lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in zip(seqs, prompts)]),
                     mode=mode, span_logits=True)
    for i, p in enumerate(prompts):
        oalloc.reserve(i, len(p))
    want_slots = np.concatenate([oalloc.slots(i, np.arange(len(p))) for i, p in enumerate(prompts)])
    assert np.array_equal(eng.last_slots, want_slots)
    e1, caches = 0.0, []
    for g, p in zip(lg, prompts):
        want, cache = torch_ref.forward(rw, p)
        e1 = max(e1, rel_err(g.cpu().numpy(), want.cpu().numpy()))
        caches.append(cache)
    tok = int(torch.argmax(lg[0][-1]))
    lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(seqs[0], [tok])]), mode=mode)
    oalloc.reserve(0, len(prompts[0]) + 1)
    assert np.array_equal(eng.last_slots, oalloc.slots(0, [len(prompts[0])]))
    want, _ = torch_ref.forward(rw, [tok], cache=caches[0])
    e2 = rel_err(lg[0].cpu().numpy(), want[0].cpu().numpy())
    # K/V of rank 5's kv head (one per rank), layer 1, vs the dense cache
    kg, vg = seqs[1].cache.read_window(5, 1, 0)
    ek = rel_err(kg.float().cpu().numpy(), caches[1].k[1][:, 5].cpu().numpy())
    ev = rel_err(vg.float().cpu().numpy(), caches[1].v[1][:, 5].cpu().numpy())
    _log(f"p8_loopback_{mode.value}", prefill=e1, decode=e2, kv=max(ek, ev))
    assert e1 <= LOGIT_TOL and e2 <= LOGIT_TOL
    assert ek <= KV_TOL and ev <= KV_TOL
