"""Speculative decoding on a B200: verify passes over
[pending, *draft] with span logits and paged rollback are token-identical to
plain greedy decoding (the reference's exactness contract,
verify_checks.py:231-261 / spec_decode.py:199-248)."""

import numpy as np
import pytest
import torch

import oracle
from oracle.model import init_weights_llama, llama_tiny_config

from helpers import c1_prompts, device_weights, rel_err

pytestmark = pytest.mark.gpu

from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy)
from paper_2507_11830_b200.spec_decode import (SpeculationConfig, decode_with_speculation,  # noqa: E402
                                               verify_and_accept)


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.fixture(scope="module")
def c1():
    return init_weights_llama(llama_tiny_config(max_seq=512), seed=0)


def _greedy_consistent(ow, prompt, out, tol=2e-2):
    """Every token of `out` is the oracle's greedy choice given the tokens
    before it, except where the oracle's top-2 margin is within the logit
    tolerance (a near-tie the bf16 path may resolve either way)."""
    for k, t in enumerate(out):
        lg, _ = oracle.forward_reference(ow, prompt + out[:k])
        row = lg[-1]
        if int(row.argmax()) != t:
            assert row.max() - row[t] <= 2 * tol * np.abs(row).max(), (k, t, int(row.argmax()))


@pytest.mark.parametrize("p,mode", [(1, None), (2, ParallelMode.TP), (2, ParallelMode.SP),
                                    (2, None)])
def test_speculation_is_token_identical_to_greedy(c1, p, mode):
    """Verify passes score every draft row in one pass (a different attention
    and GEMM row count than one-token decode), so the two runs agree token for
    token up to the first oracle near-tie, and the speculative output is a
    greedy decode throughout (teacher-forced against the oracle)."""
    eng = Engine(device_weights(c1, p), LoopbackGroup(p), ShiftPolicy(token_threshold=3))
    free0 = eng.pool.alloc.free_blocks
    prompt = [11, 42, 7, 99, 3] * 6 + c1_prompts()[2][:17]
    plain, ps = decode_with_speculation(eng, prompt, 40, SpeculationConfig(enabled=False),
                                        mode=mode)
    spec, ss = decode_with_speculation(eng, prompt, 40,
                                       SpeculationConfig(enabled=True, min_match=1, max_spec=6),
                                       mode=mode)
    assert len(plain) == len(spec) == 40
    first = next((k for k in range(40) if plain[k] != spec[k]), 40)
    assert first >= 10
    if first < 40:  # only at a near-tie
        lg, _ = oracle.forward_reference(c1, prompt + plain[:first])
        row = lg[-1]
        assert abs(row[plain[first]] - row[spec[first]]) <= 4e-2 * np.abs(row).max()
    _greedy_consistent(c1, prompt, spec)
    assert ps.target_passes == 40 and ps.drafted_total == 0
    assert ss.drafted_total > 0 and ss.accepted_total > 0 and ss.tokens_emitted == 40
    assert ss.target_passes == 1 + len(ss.accepted_lengths)
    assert ss.target_passes + ss.accepted_total == 40  # every accepted token saves a pass
    assert eng.pool.alloc.free_blocks == free0


def test_verify_rollback_keeps_cache_exact(c1):
    """A verify pass that rejects part of its draft leaves exactly the context
    plus the accepted prefix: write counter counts every staged row, the
    cursor rolls back, and the next decode matches the oracle."""
    eng = Engine(device_weights(c1, 2), LoopbackGroup(2), ShiftPolicy.fixed_tp())
    prompt = c1_prompts()[1][:24]
    s = eng.new_sequence(0, capacity=64)
    lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, prompt)]))
    pending = int(torch.argmax(lg[0]).item())
    want, _ = oracle.forward_reference(c1, prompt + [pending])
    wrong = int(want[-1].argmin())  # a draft the target must reject
    out, rec = verify_and_accept(eng, s, pending, [wrong, 5, 6], mode=ParallelMode.SP)
    assert len(out) == 1 and rec.new_tokens == 4
    assert s.cache.token_count == len(prompt) + 1
    lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, out)]), mode=ParallelMode.TP)
    want, _ = oracle.forward_reference(c1, prompt + [pending] + out)
    assert rel_err(lg[0].cpu().numpy(), want[-1]) <= 2e-2
