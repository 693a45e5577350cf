"""The fused decode layer (sp_decode_layer: one persistent kernel per layer for
the O / gate-up / down / next-QKV projections of a P = 1 TP decode pass).

Checked against the unfused kernel chain (same weights, same cache: equal up
to the f32 summation order of the K-split partials), against the fp32 oracle
(the reference algorithm, parallel_engine.py:333-398 / model.py:310-354) at
the 8B and 70B layer widths, for graph-replay == eager bit-identity and
run-to-run determinism, and at the batch edges (1, odd, 64, and 65 which falls
back to the unfused path)."""

import numpy as np
import pytest
import torch

import oracle
from oracle.model import init_weights_llama, llama_tiny_config

from helpers import device_weights, rel_err

pytestmark = pytest.mark.gpu

from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, ops)

LOGIT_TOL = 2e-2      # vs the fp32 oracle (north_star bf16 tolerance)
PATH_TOL = 1e-2       # fused vs unfused kernels: K-split points differ, so bf16
                      # roundings of xn / act / q / K / V can flip by one ulp
KV_TOL = 2 ** -7      # cached K/V are bf16: two ulps of the largest element


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def w8b():
    cfg = llama_tiny_config(n_layers=2, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336,
                            vocab_size=4096, max_seq=256)
    return init_weights_llama(cfg, seed=0)


class Spy:
    def __init__(self, monkeypatch):
        self.calls = 0
        real = ops.decode_layer

        def spy(*a, **k):
            self.calls += 1
            return real(*a, **k)
        monkeypatch.setattr(ops, "decode_layer", spy)


def _prefilled(weights, prompts, fused: bool, graphs: bool = False):
    eng = Engine(weights, LoopbackGroup(1), ShiftPolicy.fixed_tp(), cuda_graphs=graphs,
                 num_blocks=2 * len(prompts) + 16)
    eng._decode_fused = fused
    seqs = [eng.new_sequence(i, capacity=128) for i in range(len(prompts))]
    eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in zip(seqs, prompts)]),
             mode=ParallelMode.TP)
    return eng, seqs


def _prompts(b, vocab, seed=11):
    rng = np.random.default_rng(seed)
    return [[int(t) for t in rng.integers(0, vocab, size=int(rng.integers(3, 40)))]
            for _ in range(b)]


@pytest.mark.parametrize("b", [1, 5, 33, 64])
def test_fused_decode_matches_unfused_chain(w8b, b, monkeypatch):
    dw = device_weights(w8b, 1)
    prompts = _prompts(b, 4096)
    toks = [p[-1] for p in prompts]
    spy = Spy(monkeypatch)
    outs, kvs = [], []
    for fused in (False, True):
        eng, seqs = _prefilled(dw, prompts, fused)
        before = spy.calls
        lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(seqs, toks)]),
                         mode=ParallelMode.TP)
        assert (spy.calls > before) == fused  # the fused kernel ran iff enabled
        outs.append(torch.stack(lg).float().cpu().numpy())
        kvs.append([eng.pool.layer_k(0, 1).float().cpu().clone(),
                    eng.pool.layer_v(0, 1).float().cpu().clone()])
    assert rel_err(outs[1], outs[0]) <= PATH_TOL
    for a, c in zip(kvs[0], kvs[1]):   # layer-1 K/V written by the fused QKV + RoPE
        assert rel_err(c.numpy(), a.numpy()) <= KV_TOL


def test_fused_decode_vs_oracle_teacher_forced(w8b):
    dw = device_weights(w8b, 1)
    prompts = _prompts(3, 4096, seed=5)
    eng, seqs = _prefilled(dw, prompts, True)
    hist = [list(p) for p in prompts]
    rng = np.random.default_rng(2)
    for _ in range(3):
        toks = [int(t) for t in rng.integers(0, 4096, size=len(seqs))]
        lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(seqs, toks)]),
                         mode=ParallelMode.TP)
        for i, t in enumerate(toks):
            hist[i].append(t)
            want, _ = oracle.forward_reference(w8b, hist[i])
            assert rel_err(lg[i].float().cpu().numpy(), want[-1]) <= LOGIT_TOL


def test_fused_decode_70b_width_vs_oracle():
    cfg = llama_tiny_config(n_layers=1, n_heads=64, n_kv_heads=8, head_dim=128, ffn_dim=28672,
                            vocab_size=4096, max_seq=128)
    ow = init_weights_llama(cfg, seed=5)
    prompts = _prompts(3, 4096, seed=9)
    eng, seqs = _prefilled(device_weights(ow, 1), prompts, True)
    toks = [7, 4095, 0]
    lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(seqs, toks)]),
                     mode=ParallelMode.TP)
    for i, t in enumerate(toks):
        want, _ = oracle.forward_reference(ow, prompts[i] + [t])
        assert rel_err(lg[i].float().cpu().numpy(), want[-1]) <= LOGIT_TOL


def test_fused_decode_graph_replay_and_determinism(w8b):
    dw = device_weights(w8b, 1)
    prompts = _prompts(9, 4096, seed=3)
    rng = np.random.default_rng(4)
    steps = [[int(t) for t in rng.integers(0, 4096, size=9)] for _ in range(5)]
    runs = []
    for graphs in (False, True, True):
        eng, seqs = _prefilled(dw, prompts, True, graphs=graphs)
        out = []
        for toks in steps:
            lg, _ = eng.step(Batch(BatchKind.DECODE,
                                   [BatchItem(s, [t]) for s, t in zip(seqs, toks)]),
                             mode=ParallelMode.TP)
            out.append(torch.stack(lg).cpu())
        if graphs:
            entries = [e for e in eng._graphs.values() if e.graph is not None]
            assert entries and sum(e.replays for e in entries) >= 2
        runs.append(torch.stack(out))
    assert torch.equal(runs[0], runs[1])   # graph replays == eager, bit for bit
    assert torch.equal(runs[1], runs[2])   # and run to run


def test_fused_decode_batch_above_64_uses_unfused_path(w8b, monkeypatch):
    dw = device_weights(w8b, 1)
    prompts = _prompts(65, 4096, seed=8)
    spy = Spy(monkeypatch)
    eng, seqs = _prefilled(dw, prompts, True)
    lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [1]) for s in seqs]),
                     mode=ParallelMode.TP)
    assert spy.calls == 0 and len(lg) == 65


def test_decode_layer_contract_errors(w8b):
    from paper_2507_11830_b200.errors import ContractViolation
    dev = torch.device("cuda")
    x = torch.zeros((2, 4096), dtype=torch.float32, device=dev)
    xn = torch.zeros((2, 4096), dtype=torch.bfloat16, device=dev)
    w = torch.zeros((4096, 4096), dtype=torch.bfloat16, device=dev)
    sync = torch.zeros(2, dtype=torch.int32, device=dev)
    p = ops.DlProj(w, xn, ops.DL_RES_NORM, n=4096, k=4096, ldw=4096)
    ws = torch.empty(16, dtype=torch.float32, device=dev)
    with pytest.raises(ContractViolation, match="workspace"):
        ops.decode_layer(2, x, 1e-5, [p], ws=ws, sync=sync)
    big = torch.zeros((65, 4096), dtype=torch.float32, device=dev)
    with pytest.raises(ContractViolation, match="rows"):
        ops.decode_layer(65, big, 1e-5, [p], ws=ws, sync=sync)
    bad = ops.DlProj(w, xn, ops.DL_RES_NORM, n=2048, k=4096, ldw=4096)
    nb = ops.decode_layer_ws_bytes(2, x, [bad])
    ws = torch.empty(nb // 4, dtype=torch.float32, device=dev)
    with pytest.raises(ContractViolation, match="hidden wide"):
        ops.decode_layer(2, x, 1e-5, [bad], ws=ws, sync=sync)
