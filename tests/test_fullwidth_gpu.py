"""Parity at the BASELINE model widths: Llama-3.1-8B geometry
(h 4096, 32q/8kv heads of 128, f 14336, V 128256) at truncated depth (2
layers) and Llama-3.3-70B layer geometry (h 8192, 64q/8kv, f 28672) at one
layer, against the fp32 oracle on the same bf16 weights, and size-independent
properties at the full 8K bench size."""

import numpy as np
import pytest
import torch

import oracle
from oracle.model import init_weights_llama, llama_tiny_config

from helpers import device_weights, rel_err

pytestmark = pytest.mark.gpu

from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, llama31_8b)
from paper_2507_11830_b200.weights import ModelWeights  # noqa: E402

LOGIT_TOL = 2e-2


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def w8b_l2():
    cfg = llama_tiny_config(n_layers=2, n_heads=32, n_kv_heads=8, head_dim=128, ffn_dim=14336,
                            vocab_size=128256, max_seq=512)
    return init_weights_llama(cfg, seed=0)


@pytest.mark.parametrize("mode", [ParallelMode.SP, ParallelMode.TP])
def test_8b_width_prefill_and_decode_vs_oracle(w8b_l2, mode):
    rng = np.random.default_rng(3)
    prompt = [int(t) for t in rng.integers(0, 128256, size=40)]
    eng = Engine(device_weights(w8b_l2, 2), LoopbackGroup(2), ShiftPolicy.fixed_tp())
    s = eng.new_sequence(0, capacity=64)
    lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]), mode=mode,
                     span_logits=True)
    want, _ = oracle.forward_reference(w8b_l2, prompt)
    assert rel_err(lg[0].cpu().numpy(), want) <= LOGIT_TOL
    tok = int(np.argmax(want[-1]))
    lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [tok])]), mode=mode)
    want2, _ = oracle.forward_reference(w8b_l2, prompt + [tok])
    assert rel_err(lg[0].cpu().numpy(), want2[-1]) <= LOGIT_TOL


@pytest.fixture(scope="module")
def w70b_l1():
    # Llama-3.3-70B layer geometry (h 8192, 64q/8kv heads of 128, f 28672) at one
    # layer; a 4096-token vocabulary keeps the host oracle's embedding small
    cfg = llama_tiny_config(n_layers=1, n_heads=64, n_kv_heads=8, head_dim=128, ffn_dim=28672,
                            vocab_size=4096, max_seq=256)
    return init_weights_llama(cfg, seed=5)


@pytest.mark.parametrize("mode", [ParallelMode.SP, ParallelMode.TP])
def test_70b_width_prefill_and_decode_vs_oracle(w70b_l1, mode):
    """configs[3] model width: prefill (span logits) and a decode step at P=2
    against the fp32 oracle on the same bf16 weights."""
    rng = np.random.default_rng(4)
    prompt = [int(t) for t in rng.integers(0, 4096, size=24)]
    eng = Engine(device_weights(w70b_l1, 2), LoopbackGroup(2), ShiftPolicy.fixed_tp())
    s = eng.new_sequence(0, capacity=48)
    lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]), mode=mode,
                     span_logits=True)
    want, _ = oracle.forward_reference(w70b_l1, prompt)
    assert rel_err(lg[0].cpu().numpy(), want) <= LOGIT_TOL
    tok = int(np.argmax(want[-1]))
    lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [tok])]), mode=mode)
    want2, _ = oracle.forward_reference(w70b_l1, prompt + [tok])
    assert rel_err(lg[0].cpu().numpy(), want2[-1]) <= LOGIT_TOL


def test_full_8k_prefill_properties():
    """At the bench size (8B, 8192 tokens): chunked prefill reproduces the
    one-pass last-token logits within tolerance, the KV write counter equals the
    exact bytes, and logits are finite."""
    cfg = llama31_8b(n_layers=4, max_seq=8192)
    w = ModelWeights.random(cfg, seed=0, world_size=1)
    rng = np.random.default_rng(0)
    prompt = [int(t) for t in rng.integers(0, cfg.vocab_size, size=8192)]
    eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_sp(), num_blocks=300)
    a = eng.new_sequence(0, capacity=8192)
    one, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(a, prompt)]), mode=ParallelMode.SP)
    b = eng.new_sequence(1, capacity=8192)
    for lo in range(0, 8192, 2048):
        part, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(b, prompt[lo:lo + 2048])]),
                           mode=ParallelMode.SP)
    x, y = one[0].cpu().numpy(), part[0].cpu().numpy()
    assert np.all(np.isfinite(x))
    assert rel_err(y, x) <= LOGIT_TOL
    per_token = 2 * cfg.n_layers * cfg.kv_heads * cfg.head_dim * 2
    assert a.cache.write_counter == b.cache.write_counter == 8192 * per_token
