"""Interleaved A/B of the prefill-GEMM raster L2 budget (SP_GEMM_L2_MB) on the
Llama-3.1-8B projections: for every (M, projection) one CUDA graph of 10
launches per budget, captured while that budget is set, then replayed in
rounds alternating between budgets so clock/power drift hits every variant
equally.  Prints one JSON line per (M, projection): median TFLOP/s per budget.

    python tools/raster_ab.py [--budgets 40,64,100] [--rounds 7] [M ...]
"""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import ops  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--budgets", default="40,64,100")
ap.add_argument("--rounds", type=int, default=7)
ap.add_argument("Ms", nargs="*", type=int)
args = ap.parse_args()
budgets = [b for b in args.budgets.split(",")]
h, f, qkv = 4096, 14336, 6144
ops.set_gemm_workspace(torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
for M in args.Ms or [8192, 4096, 2048, 1024]:
    for name, n, k, epi in [("qkv", qkv, h, ops.EPI_STORE_BF16), ("o", h, h, ops.EPI_ADD_F32),
                            ("gate_up", 2 * f, h, ops.EPI_SWIGLU), ("down", h, f, ops.EPI_ADD_F32)]:
        a = torch.randn(M, k, device="cuda").to(torch.bfloat16)
        b = torch.randn(n, k, device="cuda").to(torch.bfloat16)
        if epi == ops.EPI_SWIGLU:
            d = torch.empty(M, n // 2, device="cuda", dtype=torch.bfloat16); ldd = n // 2
        elif epi == ops.EPI_ADD_F32:
            d = torch.zeros(M, n, device="cuda"); ldd = n
        else:
            d = torch.empty(M, n, device="cuda", dtype=torch.bfloat16); ldd = n
        graphs = {}
        s = torch.cuda.Stream()
        for bud in budgets:
            os.environ["SP_GEMM_L2_MB"] = bud
            g = torch.cuda.CUDAGraph()
            with torch.cuda.stream(s):
                ops.gemm(a, b, d, epi, M=M, N=n, K=k, lda=k, ldb=k, ldd=ldd)
                torch.cuda.synchronize()
                with torch.cuda.graph(g, stream=s):
                    for _ in range(10):
                        ops.gemm(a, b, d, epi, M=M, N=n, K=k, lda=k, ldb=k, ldd=ldd)
            g.replay()
            graphs[bud] = g
        torch.cuda.synchronize()
        ts = {bud: [] for bud in budgets}
        for rnd in range(args.rounds):
            order = budgets if rnd % 2 == 0 else budgets[::-1]
            for bud in order:
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                graphs[bud].replay()
                e1.record()
                torch.cuda.synchronize()
                ts[bud].append(e0.elapsed_time(e1) / 10)
        fl = 2 * M * n * k
        row = {"M": M, "gemm": name}
        for bud in budgets:
            ms = sorted(ts[bud])[len(ts[bud]) // 2]
            row[bud] = round(fl / ms / 1e9, 1)
        print(json.dumps(row), flush=True)
os.environ.pop("SP_GEMM_L2_MB", None)
