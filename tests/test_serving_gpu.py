"""Serving driver on a B200 with the tiny Llama (C1 weights)."""

import numpy as np
import pytest
import torch

from oracle.model import init_weights_llama, llama_tiny_config

from helpers import device_weights

pytestmark = pytest.mark.gpu

from paper_2507_11830_b200 import Engine, LoopbackGroup, ShiftPolicy  # noqa: E402
from paper_2507_11830_b200.serving import TraceEntry, run_serving, summarize  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("p", [1, 2])
def test_serving_loop_prefill_first_and_shift(p):
    ow = init_weights_llama(llama_tiny_config(max_seq=256), seed=0)
    eng = Engine(device_weights(ow, p), LoopbackGroup(p), ShiftPolicy(token_threshold=6),
                 num_blocks=64, block_size=64)
    free0 = eng.pool.alloc.free_blocks
    trace = [TraceEntry(0, 0, 40, 5), TraceEntry(1, 0, 17, 1), TraceEntry(2, 30, 33, 7),
             TraceEntry(3, 31, 9, 3), TraceEntry(4, 400, 250, 10)]  # last one is rejected
    res = run_serving(eng, trace, seed=1)
    assert [r["request_id"] for r in res.rejected] == [4]
    assert sorted(res.outputs) == [0, 1, 2, 3]
    for e in trace[:4]:
        assert len(res.outputs[e.request_id]) == e.output_len
        assert all(0 <= t < 256 for t in res.outputs[e.request_id])
    # passes never mix prefill and decode; mode follows the token threshold
    for pl in res.passes:
        assert pl.mode == ("sp" if pl.batch_tokens >= 6 else "tp")
        if pl.batch_kind == "decode":
            assert pl.batch_tokens == pl.n_requests
    assert res.passes[0].batch_kind == "prefill"
    s = summarize(res)
    assert s["requests"] == 4 and s["median_ttft_ms"] >= 0 and s["mode_shift_count"] >= 1
    assert eng.pool.alloc.free_blocks == free0  # every finished sequence released its blocks


def test_serving_admission_waits_for_blocks():
    """A pool too small for every request at once: the driver admits requests
    only while their whole lifetime fits, the rest wait for releases; all
    complete with their full outputs and the pool never overflows."""
    ow = init_weights_llama(llama_tiny_config(max_seq=256), seed=0)
    trace = [TraceEntry(i, 0, 100, 30) for i in range(6)]  # 2 blocks of 64 each
    outs = []
    for blocks in (64, 5):  # 5 blocks: at most 2 requests live
        eng = Engine(device_weights(ow, 1), LoopbackGroup(1), ShiftPolicy.fixed_tp(),
                     num_blocks=blocks, block_size=64)
        res = run_serving(eng, trace, seed=3)
        assert sorted(res.outputs) == list(range(6))
        assert eng.pool.alloc.free_blocks == blocks
        outs.append(res)
    assert max(p.n_requests for p in outs[1].passes) <= 2
    assert all(len(outs[1].outputs[i]) == 30 for i in range(6))
