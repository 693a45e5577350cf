import os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.getcwd())
from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup, ParallelMode, ShiftPolicy, llama31_8b)
from paper_2507_11830_b200.weights import ModelWeights
B, CTX = int(sys.argv[1]), 2048
cfg = llama31_8b(max_seq=CTX + 64)
w = ModelWeights.random(cfg, seed=0, world_size=1)
eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_tp(), num_blocks=B * -(-(CTX + 64) // 64) + 8)
rng = np.random.default_rng(0)
seqs = [eng.new_sequence(i, capacity=CTX + 64) for i in range(B)]
for i in range(0, B, 8):
    eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, [int(t) for t in rng.integers(0, 1000, CTX)]) for s in seqs[i:i + 8]]), mode=ParallelMode.SP)
torch.cuda.synchronize()
def step(rb):
    eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [1]) for s in seqs]), mode=ParallelMode.TP)
    if rb:
        for s in seqs: s.cache.truncate(CTX)
for rb in (True, False, True, False):
    for _ in range(4): step(rb)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for _ in range(16): step(rb)
    t1 = time.perf_counter(); e1.record(); torch.cuda.synchronize()
    print(f"B={B} rollback={rb} TPOT {e0.elapsed_time(e1)/16:.3f} ms  host {1e3*(t1-t0)/16:.3f} ms/step (enqueue)", flush=True)
if len(sys.argv) > 2 and sys.argv[2] == "prof":
    import cProfile, pstats
    pr = cProfile.Profile()
    pr.enable()
    for _ in range(16): step(False)
    torch.cuda.synchronize()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(18)
