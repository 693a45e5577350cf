"""Pin the torch fp32 checker (tests/torch_ref.py) to the numpy oracle on the
CPU, so the GPU parity tests at the BASELINE shapes stay chained to the
reference: oracle == shiftsim (bit-exact, test_oracle_golden.py) and
torch_ref == oracle (here)."""

import numpy as np
import pytest
import torch

import oracle
from oracle.model import compat_config, init_weights_compat, init_weights_llama, llama_tiny_config

import torch_ref
from helpers import host_dict, product_config, rel_err


def _prompt(seed, n, vocab):
    return [int(t) for t in np.random.default_rng(seed).integers(0, vocab, size=n)]


@pytest.fixture(scope="module")
def tiny():
    return init_weights_llama(llama_tiny_config(max_seq=256), seed=0)


@pytest.mark.parametrize("emulate", [False, True])
def test_llama_prefill_and_continuation_match_oracle(tiny, emulate):
    rw = torch_ref.RefWeights.from_oracle(tiny)
    p = _prompt(1, 57, 256)
    want, ocache = oracle.forward_reference(tiny, p, emulate_bf16=emulate)
    got, cache = torch_ref.forward(rw, p, emulate_bf16=emulate)
    # fp32 with different summation orders; with bf16 emulation a rounding
    # boundary may flip one stored bf16 value
    tol = 5e-3 if emulate else 2e-5
    assert rel_err(got.numpy(), want) <= tol
    want2, _ = oracle.forward_reference(tiny, [3, 9], cache=ocache, emulate_bf16=emulate)
    got2, _ = torch_ref.forward(rw, [3, 9], cache=cache, emulate_bf16=emulate)
    assert rel_err(got2.numpy(), want2) <= tol


def test_logit_rows_and_hidden(tiny):
    rw = torch_ref.RefWeights.from_oracle(tiny)
    p = _prompt(2, 40, 256)
    full, _ = torch_ref.forward(rw, p)
    hid = {}
    some, _ = torch_ref.forward(rw, p, logit_rows=[0, 39], hidden_out=hid)
    assert torch.allclose(some, full[[0, 39]], rtol=1e-5, atol=1e-6)
    assert hid["x"].shape == (2, 256)


def test_compat_f64_matches_oracle():
    """The reference's own family (MHA, sinusoidal, GeLU, eps 1e-6) in f64."""
    cfg = compat_config(n_layers=2, n_heads=4, head_dim=16, ffn_dim=128, vocab_size=64,
                        max_seq=128)
    ow = init_weights_compat(cfg, seed=3)
    rw = torch_ref.RefWeights.from_oracle(ow, dtype=torch.float64)
    p = _prompt(4, 30, 64)
    want, _ = oracle.forward_reference(ow, p)
    got, _ = torch_ref.forward(rw, p)
    assert rel_err(got.numpy(), want) <= 1e-12


def test_swiftkv_matches_oracle_engine(tiny):
    oeng = oracle.OracleEngine(tiny, 1, swiftkv_cut=2)
    s = oeng.new_sequence(0, capacity=96)
    p = _prompt(5, 77, 256)
    olg, _ = oeng.step([(s, p)], mode="tp")
    got, _ = torch_ref.forward_swiftkv(torch_ref.RefWeights.from_oracle(tiny), p, cut=2)
    assert rel_err(got[0].numpy(), olg[0]) <= 2e-5


@pytest.mark.parametrize("world", [1, 2, 8])
def test_from_model_undoes_product_layouts(tiny, world):
    """The product's fused / permuted device layouts (per-rank q|k|v rows,
    gate/up interleave) map back to exactly the oracle's matrices."""
    from paper_2507_11830_b200.weights import ModelWeights
    if world == 8:  # one kv head per rank, as 8B at P=8
        tiny = init_weights_llama(llama_tiny_config(n_kv_heads=8, max_seq=256), seed=2)
    cfg = product_config(tiny.config)
    mw = ModelWeights.from_host(cfg, host_dict(tiny), world, device="cpu")
    a = torch_ref.RefWeights.from_model(mw)
    b = torch_ref.RefWeights.from_oracle(tiny)
    for li in (0, 3):
        la, lb = a.layer(li), b.layer(li)
        for k in lb:
            assert torch.equal(la[k], lb[k]), (li, k)
    p = _prompt(6, 20, 256)
    ga, _ = torch_ref.forward(a, p)
    gb, _ = torch_ref.forward(b, p)
    assert torch.equal(ga, gb)
