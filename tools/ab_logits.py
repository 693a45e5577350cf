"""Bit-identity A/B between two library builds: the same 8B-geometry engine
(2 layers, random weights) runs a prefill and decode steps at several batch
sizes; logits are saved per run and compared.

    SP_LIB_PATH=<lib A> python tools/ab_logits.py save /tmp/a.pt
    SP_LIB_PATH=<lib B> python tools/ab_logits.py save /tmp/b.pt
    python tools/ab_logits.py compare /tmp/a.pt /tmp/b.pt
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def save(path):
    from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,
                                       ParallelMode, ShiftPolicy, llama31_8b)
    from paper_2507_11830_b200.weights import ModelWeights
    out = {}
    for B, ctx in ((1, 2048), (4, 1000), (16, 300), (64, 700)):
        cfg = llama31_8b(max_seq=ctx + 64, n_layers=2)
        w = ModelWeights.random(cfg, seed=0, world_size=1)
        eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_tp(), num_blocks=B * -(-(ctx + 64) // 64) + 8)
        rng = np.random.default_rng(B)
        seqs = [eng.new_sequence(i, capacity=ctx + 64) for i in range(B)]
        lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, [int(t) for t in rng.integers(0, 1000, ctx)])
                                                   for s in seqs]), mode=ParallelMode.SP)
        out[f"b{B}_prefill"] = lg[0].float().cpu() if isinstance(lg, list) else lg.float().cpu()
        for step in range(4):  # eager, capture, replays
            lg, _ = eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [int(rng.integers(0, 1000))]) for s in seqs]),
                             mode=ParallelMode.TP)
            out[f"b{B}_decode{step}"] = torch.stack([x.float().cpu() for x in lg]) if isinstance(lg, list) \
                else lg.float().cpu()
        del eng, w
        torch.cuda.empty_cache()
    torch.save(out, path)
    print(f"saved {len(out)} logit sets to {path}")


def compare(a, b):
    A, Bd = torch.load(a), torch.load(b)
    bad = 0
    for k in A:
        same = torch.equal(A[k], Bd[k])
        bad += not same
        print(f"{k:18s} {'identical' if same else 'DIFFERENT max|d|=%.3g' % (A[k] - Bd[k]).abs().max()}")
    print("ALL IDENTICAL" if bad == 0 else f"{bad} sets differ")


if __name__ == "__main__":
    if sys.argv[1] == "save":
        save(sys.argv[2])
    else:
        compare(sys.argv[2], sys.argv[3])
