"""One 8B decode setup (B requests at ctx), then graph-replayed decode steps.
Run under `ncu --metrics gpu__time_duration.sum` to get per-kernel device
times of a decode step (graph nodes are profiled individually).

    python tools/decode_profile.py [B] [ctx] [steps]
"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, llama31_8b)
from paper_2507_11830_b200.weights import ModelWeights  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
CTX = int(sys.argv[2]) if len(sys.argv) > 2 else 2048
STEPS = int(sys.argv[3]) if len(sys.argv) > 3 else 3
torch.cuda.set_device(0)
cfg = llama31_8b(max_seq=CTX + 64)
w = ModelWeights.random(cfg, seed=0, world_size=1)
eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_tp(), num_blocks=B * -(-(CTX + 64) // 64) + 8)
rng = np.random.default_rng(0)
seqs = [eng.new_sequence(i, capacity=CTX + 64) for i in range(B)]
for i in range(0, B, 8):
    eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, [int(t) for t in rng.integers(0, 1000, CTX)])
                                       for s in seqs[i:i + 8]]), mode=ParallelMode.SP)
torch.cuda.synchronize()
for step in range(STEPS + 2):
    eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [1]) for s in seqs]), mode=ParallelMode.TP)
torch.cuda.synchronize()
s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s0.record()
for step in range(STEPS):
    eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [1]) for s in seqs]), mode=ParallelMode.TP)
s1.record()
torch.cuda.synchronize()
print(f"B={B} ctx={CTX} TPOT {s0.elapsed_time(s1) / STEPS:.3f} ms")
