"""Prefill-GEMM throughput at the per-GPU token counts of SP strong scaling
(8K tokens over N GPUs -> M = 8192/N), Llama-3.1-8B projection shapes.

    [SP_GEMM_2CTA=0] [SP_GEMM_FORCE_BN=128] python tools/gemm_sweep.py [M ...]
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import ops  # noqa: E402

h, f, qkv = 4096, 14336, 6144
Ms = [int(x) for x in sys.argv[1:]] or [1024, 2048, 4096, 8192]
ops.set_gemm_workspace(torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
for M in Ms:
    row = {"M": M}
    tot_ms, tot_fl = 0.0, 0
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
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            ops.gemm(a, b, d, epi, M=M, N=n, K=k, lda=k, ldb=k, ldd=ldd)
            torch.cuda.synchronize()
            with torch.cuda.graph(g, stream=s):
                for _ in range(10):
                    ops.gemm(a, b, d, epi, M=M, N=n, K=k, lda=k, ldb=k, ldd=ldd)
        g.replay()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            g.replay()
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / 10)
        ms = sorted(ts)[2]
        fl = 2 * M * n * k
        row[name] = round(fl / ms / 1e9, 1)
        tot_ms += ms
        tot_fl += fl
    row["layer_tflops"] = round(tot_fl / tot_ms / 1e9, 1)
    print(json.dumps(row), flush=True)
