"""Host-side cost of one 8K prefill through Engine.step (the e2e path):
wall time of the call (launches are asynchronous), the D2H wait, and a
cProfile of the host work.

    python tools/prefill_host_probe.py
"""
import cProfile
import os
import pstats
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, llama31_8b)
from paper_2507_11830_b200.weights import ModelWeights  # noqa: E402

S = 8192
cfg = llama31_8b(max_seq=S)
w = ModelWeights.random(cfg, seed=0, world_size=1)
eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_sp(), num_blocks=S // 64 + 8, block_size=64)
prompt = [int(t) for t in np.random.default_rng(0).integers(0, cfg.vocab_size, size=S)]
seq = eng.new_sequence(0, capacity=S)


def one():
    seq.cache.truncate(0)
    t0 = time.perf_counter()
    lg, _ = eng.step(Batch(BatchKind.PREFILL, [BatchItem(seq, prompt)]), mode=ParallelMode.SP)
    t1 = time.perf_counter()
    h = lg[0].cpu()
    t2 = time.perf_counter()
    return t1 - t0, t2 - t1


for _ in range(3):
    one()
torch.cuda.synchronize()
for _ in range(3):
    a, b = one()
    print(f"step() returns after {a * 1e3:.2f} ms, logits ready {b * 1e3:.2f} ms later, total {(a + b) * 1e3:.2f} ms")
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record()
seq.cache.truncate(0)
eng.step(Batch(BatchKind.PREFILL, [BatchItem(seq, prompt)]), mode=ParallelMode.SP)
e1.record()
torch.cuda.synchronize()
print(f"device time of one step {e0.elapsed_time(e1):.2f} ms")
e0.record()
for _ in range(3):
    seq.cache.truncate(0)
    eng.step(Batch(BatchKind.PREFILL, [BatchItem(seq, prompt)]), mode=ParallelMode.SP)
e1.record()
torch.cuda.synchronize()
print(f"device time per step, 3 back to back {e0.elapsed_time(e1) / 3:.2f} ms")
# host time from step() entry to the first kernel launch (the embedding)
from paper_2507_11830_b200 import ops  # noqa: E402
stamp = {}
_embed = ops.embed


def embed_stamp(*a, **k):
    stamp.setdefault("t", time.perf_counter())
    return _embed(*a, **k)


ops.embed = embed_stamp
import paper_2507_11830_b200.engine as engmod  # noqa: E402
engmod.ops.embed = embed_stamp
for _ in range(3):
    stamp.clear()
    torch.cuda.synchronize()
    seq.cache.truncate(0)
    t0 = time.perf_counter()
    eng.step(Batch(BatchKind.PREFILL, [BatchItem(seq, prompt)]), mode=ParallelMode.SP)
    print(f"step() entry -> first launch {(stamp['t'] - t0) * 1e3:.3f} ms")
torch.cuda.synchronize()
ops.embed = _embed
engmod.ops.embed = _embed
pr = cProfile.Profile()
pr.enable()
one()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(40)
