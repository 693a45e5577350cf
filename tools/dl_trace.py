"""Timeline of one fused decode-layer launch (sp_decode_layer, -DDL_TRACE build).

Builds paper_2507_11830_b200/libshiftpar_trace.so with -DDL_TRACE (if absent,
here — needs nvcc), runs an 8B decode step (eager, P = 1, TP) and prints, per
instrumented milestone, the min / median / max over CTAs of its globaltimer
stamp relative to the earliest stamp of the launch (microseconds).

    python tools/dl_trace.py [B] [ctx] [call]      # call: which launch of the step (default 6)
"""
import ctypes
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2507_11830_b200", "libshiftpar_trace.so")
if __name__ == "__main__" and not os.path.exists(LIB):
    sys.path.insert(0, ROOT)
    from paper_2507_11830_b200 import build as b
    subprocess.run([os.environ.get("NVCC", "nvcc"), *b.NVCC_FLAGS, "-DDL_TRACE", "-I",
                    os.path.join(ROOT, "include"), "-o", LIB, *b.sources()], check=True)
os.environ["SP_LIB_PATH"] = LIB
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2507_11830_b200 import (Batch, BatchItem, BatchKind, Engine, LoopbackGroup,  # noqa: E402
                                   ParallelMode, ShiftPolicy, _lib, llama31_8b, ops)
from paper_2507_11830_b200.weights import ModelWeights  # noqa: E402

NAMES = {0: "epilogue start", 1: "first weight box", 2: "predecessor wait done"}
for p in range(4):
    NAMES[3 + p] = f"proj{p} input ready"
    NAMES[7 + p] = f"proj{p} first MMA"
    NAMES[11 + p] = f"proj{p} last MMA issued"
    NAMES[15 + p] = f"proj{p} partials written"
NAMES.update({40: "CTA0 norm start", 41: "CTA0 norm x loaded", 42: "CTA0 norm sum done",
              43: "CTA0 norm stored", 45: "CTA0 swiglu start", 46: "CTA0 swiglu gate sum",
              47: "CTA0 swiglu up sum", 49: "CTA0 swiglu stored", 50: "probe seg0 ld", 51: "probe seg1 ld",
              52: "probe seg2 ld", 53: "probe seg1 ld again", 54: "probe owner math"})
for k in range(10):
    NAMES[20 + 2 * k] = f"barrier {k + 1} arrive"
    NAMES[21 + 2 * k] = f"barrier {k + 1} pass"


def main():
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 1
    CTX = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    CALL = int(sys.argv[3]) if len(sys.argv) > 3 else 6
    REPEAT = os.environ.get("DL_TRACE_REPEAT") == "1"  # trace an immediate re-launch (warm code)
    torch.cuda.set_device(0)
    cfg = llama31_8b(max_seq=CTX + 64)
    w = ModelWeights.random(cfg, seed=0, world_size=1)
    eng = Engine(w, LoopbackGroup(1), ShiftPolicy.fixed_tp(), cuda_graphs=False,
                 num_blocks=B * -(-(CTX + 64) // 64) + 8)
    rng = np.random.default_rng(0)
    seqs = [eng.new_sequence(i, capacity=CTX + 64) for i in range(B)]
    for i in range(0, B, 8):
        eng.step(Batch(BatchKind.PREFILL, [BatchItem(s, [int(t) for t in rng.integers(0, 1000, CTX)])
                                           for s in seqs[i:i + 8]]), mode=ParallelMode.SP)
    lib = _lib.load()
    lib.sp_decode_layer_trace.restype = ctypes.c_int
    lib.sp_decode_layer_trace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    real = ops.decode_layer
    state = {"n": 0, "trace": None}

    def spy(*a, **k):
        real(*a, **k)
        state["n"] += 1
        if state["n"] == CALL:
            if REPEAT:
                real(*a, **k)
            buf = (ctypes.c_ulonglong * (160 * 64))()
            torch.cuda.synchronize()
            lib.sp_decode_layer_trace(buf, 160 * 64)
            state["trace"] = np.frombuffer(buf, dtype=np.uint64).reshape(160, 64).astype(np.int64)
    ops.decode_layer = spy
    for _ in range(2):
        state["n"] = 0
        eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [1]) for s in seqs]), mode=ParallelMode.TP)
    # kernel-level timeline of one more (eager) step: start / end of every fused launch
    lib.sp_decode_layer_ktrace.restype = ctypes.c_int
    lib.sp_decode_layer_ktrace.argtypes = [ctypes.c_void_p, ctypes.c_int]
    lib.sp_decode_layer_ktrace(None, 1)
    ops.decode_layer = real
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    eng.step(Batch(BatchKind.DECODE, [BatchItem(s, [1]) for s in seqs]), mode=ParallelMode.TP)
    e1.record()
    kt = (ctypes.c_ulonglong * 1024)()
    n = lib.sp_decode_layer_ktrace(kt, 0)
    kt = np.frombuffer(kt, dtype=np.uint64).reshape(512, 2).astype(np.int64)[:n]
    print(f"eager step {e0.elapsed_time(e1):.3f} ms; {n} fused launches")
    dur = (kt[:, 1] - kt[:, 0]) / 1e3
    gap = (kt[1:, 0] - kt[:-1, 1]) / 1e3
    print(f"fused launch duration us: median {np.median(dur):.1f} min {dur.min():.1f} max {dur.max():.1f}")
    print(f"gap end->next start us:   median {np.median(gap):.1f} min {gap.min():.1f} max {gap.max():.1f}")
    print(f"first start -> last end: {(kt[-1, 1] - kt[0, 0]) / 1e3:.1f} us")
    tr = state["trace"]
    G = eng._sms
    tr = tr[:G]
    valid = tr > 0
    t0 = tr[valid].min()
    print(f"B={B} ctx={CTX} launch #{CALL} of the step, {G} CTAs; us from the first stamp")
    print(f"{'milestone':28s} {'min':>8s} {'median':>8s} {'max':>8s}  n")
    for s in range(64):
        col = tr[:, s]
        col = col[col > 0]
        if len(col) == 0:
            continue
        us = (col - t0) / 1e3
        print(f"{NAMES.get(s, str(s)):28s} {us.min():8.2f} {np.median(us):8.2f} {us.max():8.2f}  {len(col)}")


if __name__ == "__main__":
    main()
