"""In-graph cost of each kernel class of a decode step (ablation: the class is
replaced by a no-op and the CUDA-graph TPOT re-measured; results are NOT valid
outputs — timing analysis only).

    python tools/decode_ablation.py [B] [ctx]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, llama31_8b, ops)
from paper_2507_11830_b200.weights import ModelWeights  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
CTX = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
cfg = llama31_8b(max_seq=CTX + 64)
w = ModelWeights.random(cfg, seed=0, world_size=1)
orig = {k: getattr(ops, k) for k in ("gemm", "attention", "attention_decode_qkv", "add_rmsnorm",
                                     "rope_kv_write", "rope_kv_write_partials")}


def run(label, skip):
    for k, f in orig.items():
        setattr(ops, k, f)
    if skip:
        def gemm(a, b, d, epi, *, M, N, K, **kw):
            if (N, K) in skip.get("gemm", ()):
                return
            return orig["gemm"](a, b, d, epi, M=M, N=N, K=K, **kw)
        ops.gemm = gemm
        for k in ("attention", "attention_decode_qkv", "add_rmsnorm", "rope_kv_write",
                  "rope_kv_write_partials"):
            if k in skip:
                setattr(ops, k, lambda *a, **kw: None)
    eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_tp(), num_blocks=B * -(-(CTX + 64) // 64) + 8)
    rng = np.random.default_rng(0)
    seqs = [eng.new_sequence(i, capacity=CTX + 64) for i in range(B)]
    for s in seqs:  # context via a cheap fake: commit tokens without computing them
        s.cache.token_count  # noqa: B018
    for i in range(0, B, 8):
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, [int(t) for t in rng.integers(0, 1000, CTX)])
                                           for s in seqs[i:i + 8]]), mode=ParallelMode.SP)

    def dstep():
        eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [1]) for s in seqs]), mode=ParallelMode.TP)
        for s in seqs:
            s.cache.truncate(s.cache.token_count - 1)

    for _ in range(4):
        dstep()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dstep()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"{label:28s} TPOT {ms:7.3f} ms", flush=True)
    del eng
    torch.cuda.empty_cache()
    return ms


h, f, W = cfg.hidden, cfg.ffn_dim, w.qkv_width
base = run("baseline", None)
if len(sys.argv) > 3 and sys.argv[3] == "base":
    sys.exit(0)
# decode passes run RoPE + the KV write inside the attention kernel
# (attention_decode_qkv) unless SP_FUSE_ATTN_ROPE=0: the attention row then
# covers both and the rope row is empty
for label, skip in [("- attention (+rope/kv)", {"attention": 1, "attention_decode_qkv": 1}),
                    ("- qkv gemm", {"gemm": [(W, h)]}),
                    ("- o gemm", {"gemm": [(h, cfg.n_heads * cfg.head_dim)]}),
                    ("- gate_up gemm", {"gemm": [(2 * f, h)]}),
                    ("- down gemm", {"gemm": [(h, f)]}),
                    ("- lm head", {"gemm": [(cfg.vocab_size, h)]}),
                    ("- norms", {"add_rmsnorm": 1}),
                    ("- rope/kv write", {"rope_kv_write": 1, "rope_kv_write_partials": 1})]:
    ms = run(label, skip)
    print(f"{'':28s} -> class costs {base - ms:7.3f} ms/step ({(base - ms) / 32 * 1e3:6.1f} us/layer)")
