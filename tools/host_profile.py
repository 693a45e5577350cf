"""Host-side cost of Engine.step for graph-replayed decode passes (cProfile).

    python tools/host_profile.py [B] [ctx] [layers]
"""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, llama31_8b)
from paper_2507_11830_b200.weights import ModelWeights  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
CTX = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
L = int(sys.argv[3]) if len(sys.argv) > 3 else 32
cfg = llama31_8b(max_seq=CTX + 64, n_layers=L)
w = ModelWeights.random(cfg, seed=0, world_size=1)
eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_tp(), num_blocks=B * -(-(CTX + 64) // 64) + 8)
rng = np.random.default_rng(0)
seqs = [eng.new_sequence(i, capacity=CTX + 64) for i in range(B)]
for i in range(0, B, 8):
    eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, [int(t) for t in rng.integers(0, 1000, CTX)])
                                       for s in seqs[i:i + 8]]), mode=ParallelMode.SP)


def dstep():
    return eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [1]) for s in seqs]), mode=ParallelMode.TP)


for _ in range(3):
    dstep()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
recs = [dstep()[1] for _ in range(20)]
torch.cuda.synchronize()
pr.disable()
print(f"B={B} layers={L} host_ms per step: {[round(r.host_ms, 3) for r in recs[-5:]]}")
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
