"""Host-side pieces of the operator-level drop-in (no GPU needed): contract
errors raised before any device work (and no CPU fallback), the
reference-shaped DeviceGroup's data-movement collectives and ledger, and the
model/flops API functions (tp_shard_view, check_shard_containment,
memory_report, swiftkv_flop_ratio) — against the reference itself when it is
importable (build container: /root/reference; GPU box: baseline/_ref)."""

import os
import sys

import numpy as np
import pytest
import torch

from oracle.model import init_weights_llama, llama_tiny_config

from helpers import host_dict, product_config

from paper_2507_11830_b200 import (check_shard_containment, collectives, llama31_8b,
                                   memory_report, swiftkv_flop_ratio, tensor_core as tc,
                                   tp_shard_view)
from paper_2507_11830_b200.config import ModelConfig
from paper_2507_11830_b200.errors import ContractViolation
from paper_2507_11830_b200.weights import ModelWeights

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _shiftsim():
    for path in (os.path.join(ROOT, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(path, "shiftsim")):
            if path not in sys.path:
                sys.path.insert(0, path)
            import shiftsim
            return shiftsim
    pytest.skip("reference package not importable here")


def test_contract_errors_before_device_work():
    a = np.ones((3, 4))
    for bad in ((np.ones((2, 3, 4)), a), (a, np.ones((5, 2))), (a.astype(np.float16), a.T)):
        with pytest.raises(ContractViolation):
            tc.matmul(*bad)
    with pytest.raises(ContractViolation):
        tc.attend_cached(np.ones((3, 16)), np.ones((5, 16)), np.ones((5, 16)), 1)
    with pytest.raises(ContractViolation):
        tc.rms_norm(np.ones((2, 8)), np.ones(4))
    with pytest.raises(ContractViolation):
        tc.sinusoidal_positions([0, 1], 7)


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    """Valid operands without a CUDA device raise; nothing computes on the host."""
    with pytest.raises(ContractViolation):
        tc.matmul(np.ones((2, 3)), np.ones((3, 4)))
    with pytest.raises(ContractViolation):
        collectives.DeviceGroup(2).all_reduce_sum([np.ones(3), np.ones(3)])


def test_sinusoidal_matches_reference():
    ss = _shiftsim()
    from shiftsim.tensor_core import sinusoidal_positions as ref
    assert np.array_equal(tc.sinusoidal_positions([0, 5, 77], 64), ref([0, 5, 77], 64))


def test_device_group_movement_and_ledger_match_reference():
    ss = _shiftsim()
    ours, theirs = collectives.DeviceGroup(3), ss.DeviceGroup(3)
    blocks = [[np.full((r + 1, 4), 10.0 * s + r) for r in range(3)] for s in range(3)]
    a, b = ours.all_to_all(blocks), theirs.all_to_all(blocks)
    assert all(np.array_equal(x, y) for ra, rb in zip(a, b) for x, y in zip(ra, rb))
    shards = [np.ones((2, 4)) * r for r in range(3)]
    assert np.array_equal(ours.all_gather(shards), theirs.all_gather(shards))
    ours.broadcast(2, np.ones(8))
    theirs.broadcast(2, np.ones(8))
    with pytest.raises(ContractViolation):
        ours.all_to_all(blocks[:2])
    assert [(r.kind.value, r.device, r.bytes, r.event_id) for r in ours.records] == \
        [(r.kind.value, r.device, r.bytes, r.event_id) for r in theirs.records]
    assert {d: {k.value: v for k, v in x.items()} for d, x in ours.ledger().items()} == \
        {d: {k.value: v for k, v in x.items()} for d, x in theirs.ledger().items()}
    assert ours.map_ranks(lambda r: r * r) == [0, 1, 4]


def test_memory_report_and_swiftkv_ratio_match_reference():
    ss = _shiftsim()
    rc = ss.ModelConfig()
    ours = ModelConfig(n_layers=rc.n_layers, n_heads=rc.n_heads, head_dim=32, ffn_dim=rc.ffn_dim,
                       vocab_size=rc.vocab_size, max_seq=rc.max_seq)  # reference family (MHA, GeLU)
    rc = ss.ModelConfig(head_dim=32)
    want = ss.memory_report(rc, 4)
    got = memory_report(ours, 4)
    assert {k: got[k] for k in want} == want
    from shiftsim.swiftkv import swiftkv_flop_ratio as ref_ratio
    for n, cut in ((64, None), (256, 1), (300, 3)):
        assert swiftkv_flop_ratio(ours, n, cut) == pytest.approx(ref_ratio(rc, n, cut), rel=1e-12)


def test_8b_report_and_ratio():
    r = memory_report(llama31_8b(), 8)
    assert r["sharded_ratio"] == 8 and r["kv_bytes_per_token_per_device"] == 16384
    assert abs(r["replica_bytes_per_device"] / 2 ** 30 - 14.96) < 0.01
    assert 0.50 <= swiftkv_flop_ratio(llama31_8b(), 32768, 16) <= 0.52


@pytest.mark.parametrize("world", [1, 2])
def test_tp_shard_views_are_contained(world):
    ow = init_weights_llama(llama_tiny_config(max_seq=128), seed=0)
    w = ModelWeights.from_host(product_config(ow.config), host_dict(ow), world, device="cpu")
    assert check_shard_containment(w)
    sh = tp_shard_view(w, world - 1)
    W = w.qkv_width
    assert torch.equal(sh.layers[0].wqkv, w.layers[0].wqkv[(world - 1) * W:world * W])
    assert sh.layers[0].wo.data_ptr() - w.layers[0].wo.data_ptr() == \
        (world - 1) * (8 // world) * 32 * 2
    with pytest.raises(ContractViolation):
        tp_shard_view(w, world)
