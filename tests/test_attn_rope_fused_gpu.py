"""Decode attention fed by the QKV K-split partials (sp_attention_decode_qkv:
RoPE + the new token's paged KV write inside the TMA decode attention kernel)
is bit-identical to the two-kernel path it replaces (sp_rope_kv_write_partials
then sp_attention) — outputs and the written K/V pages — at the kernel level
(single and many KV splits, pages of 64 and 128, GQA groups 4 and 8) and
through the engine (TP decode at P = 1 and 2, eager and graph-replayed).
Reference: kv_cache.append (kv_cache.py:99-122) + attend_cached
(tensor_core.py:135-176) of one decode layer (parallel_engine.py:359-368)."""

import numpy as np
import pytest
import torch

from oracle.model import init_weights_llama, llama_tiny_config

from helpers import device_weights

pytestmark = pytest.mark.gpu

from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, ops)
from paper_2507_11830_b200.weights import rope_table  # noqa: E402


@pytest.fixture(scope="module", autouse=True)
def _dev():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("B,ctx,hq,hk,bs,n_parts", [
    (1, 2048, 32, 8, 64, 7),      # many KV splits, the new token in the last split
    (5, 333, 32, 8, 128, 3),      # ragged contexts, 128-key pages
    (64, 900, 32, 8, 64, 7),      # one split per (item, kv head)
    (3, 1500, 64, 8, 64, 5),      # 70B-style group of 8
])
@pytest.mark.parametrize("tc", ["0", "1"])
def test_decode_qkv_kernel_bitexact(B, ctx, hq, hk, bs, n_parts, tc, monkeypatch):
    monkeypatch.setenv("SP_DECODE_TC", tc)  # mma.sync or tcgen05/TMEM decode consumers
    torch.manual_seed(B * 7 + ctx)
    d = 128
    W = (hq + 2 * hk) * d
    g = torch.Generator(device="cuda").manual_seed(ctx)
    lens = [ctx - 37 * i % 200 for i in range(B)]       # kv_len of each item (incl. the new token)
    nb = [-(-n // bs) for n in lens]
    nblk = sum(nb) + 4
    k0 = (torch.randn(nblk, hk, bs, d, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    v0 = (torch.randn(nblk, hk, bs, d, device="cuda", generator=g) * 0.5).to(torch.bfloat16)
    width = max(nb)
    bt = torch.zeros(B, width, dtype=torch.int32)
    perm = torch.randperm(nblk - 4)
    off = 0
    for i, n in enumerate(nb):
        bt[i, :n] = perm[off:off + n]
        off += n
    bt = bt.cuda()
    kvl = torch.tensor(lens, dtype=torch.int32, device="cuda")
    pos = kvl - 1
    slot = torch.tensor([int(bt[i, (lens[i] - 1) // bs]) * bs + (lens[i] - 1) % bs for i in range(B)],
                        dtype=torch.int32, device="cuda")
    cu = torch.arange(B + 1, dtype=torch.int32, device="cuda")
    parts = torch.randn(n_parts, B, W, device="cuda", generator=g) * 0.3
    rope = torch.from_numpy(rope_table(max(lens) + 8, 128, 500000.0, None)).cuda()
    ws = torch.empty(ops.attn_workspace_bytes(B, hq, d, max(lens)) // 4, device="cuda")
    # reference: the two-kernel path
    ka, va = k0.clone(), v0.clone()
    q = torch.empty(B, hq * d, dtype=torch.bfloat16, device="cuda")
    ops.rope_kv_write_partials(parts, n_parts, pos, slot, rope, q, ka, va, rows=B, q_heads=hq,
                               kv_heads=hk, head_dim=d, block_size=bs)
    oa = torch.empty(B, hq * d, dtype=torch.bfloat16, device="cuda")
    ops.attention(q, ka, va, bt, cu, pos, kvl, oa, n_items=B, work=None, n_work=0, max_q_len=1,
                  max_kv_len=max(lens), q_heads=hq, kv_heads=hk, head_dim=d, block_size=bs, ws=ws)
    # fused
    kb, vb = k0.clone(), v0.clone()
    ob = torch.empty_like(oa)
    ops.attention_decode_qkv(parts, n_parts, pos, slot, rope, kb, vb, bt, cu, kvl, ob, n_items=B,
                             max_kv_len=max(lens), q_heads=hq, kv_heads=hk, block_size=bs, ws=ws)
    torch.cuda.synchronize()
    assert torch.equal(ka, kb) and torch.equal(va, vb)
    assert torch.equal(oa, ob)


@pytest.mark.parametrize("P", [1, 2])
def test_engine_decode_fused_attention_bitexact(P):
    cfg = llama_tiny_config(n_layers=2, n_heads=8, n_kv_heads=4, head_dim=128, ffn_dim=2048,
                            vocab_size=512, max_seq=256)
    ow = init_weights_llama(cfg, seed=3)
    rng = np.random.default_rng(1)
    prompts = [[int(t) for t in rng.integers(0, 512, size=int(rng.integers(5, 60)))]
               for _ in range(6)]
    steps = [[int(t) for t in rng.integers(0, 512, size=6)] for _ in range(4)]
    runs = []
    for fused, graphs in ((False, False), (True, False), (True, True)):
        eng = Engine(device_weights(ow, P), LoopbackGroup(P), ShiftPolicy.fixed_tp(),
                     cuda_graphs=graphs)
        eng._fuse_attn_rope = fused
        seqs = [eng.new_sequence(i, capacity=128) for i in range(6)]
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, p) for s, p in zip(seqs, prompts)]),
                 mode=ParallelMode.TP)
        out = []
        for toks in steps:
            lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [t]) for s, t in zip(seqs, toks)]),
                             mode=ParallelMode.TP)
            out.append(torch.stack(lg).cpu())
        pool = [eng.pool.layer_k(r, 1).cpu().clone() for r in range(P)]
        runs.append((torch.stack(out), pool))
    for other in runs[1:]:
        assert torch.equal(runs[0][0], other[0])
        for a, b in zip(runs[0][1], other[1]):
            assert torch.equal(a, b)

