"""One eager launch of each Llama-3.1-8B prefill projection (QKV, O, gate/up,
down) at M tokens, for an ncu DRAM-traffic capture per GEMM:

    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --clock-control none --csv --log-file X.csv python tools/gemm_traffic.py [M]

Prints the algorithmic bytes of each launch (A + B read once, C written once,
+ C read for the residual-add epilogues) so the capture can be divided by it.
Raster knobs (SP_GEMM_RASTER=m|n, SP_GEMM_L2_MB) apply as in the engine.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import ops  # noqa: E402

h, f, qkv = 4096, 14336, 6144
M = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
ops.set_gemm_workspace(torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
out = {}
for name, n, k, epi in [("qkv", qkv, h, ops.EPI_STORE_BF16), ("o", h, h, ops.EPI_ADD_F32),
                        ("gate_up", 2 * f, h, ops.EPI_SWIGLU), ("down", h, f, ops.EPI_ADD_F32)]:
    a = torch.randn(M, k, device="cuda").to(torch.bfloat16)
    b = torch.randn(n, k, device="cuda").to(torch.bfloat16)
    if epi == ops.EPI_SWIGLU:
        d = torch.empty(M, n // 2, device="cuda", dtype=torch.bfloat16)
        ldd, c_bytes = n // 2, M * (n // 2) * 2
    elif epi == ops.EPI_ADD_F32:
        d = torch.zeros(M, n, device="cuda")
        ldd, c_bytes = n, 2 * M * n * 4
    else:
        d = torch.empty(M, n, device="cuda", dtype=torch.bfloat16)
        ldd, c_bytes = n, M * n * 2
    torch.cuda.synchronize()
    ops.gemm(a, b, d, epi, M=M, N=n, K=k, lda=k, ldb=k, ldd=ldd)
    torch.cuda.synchronize()
    out[name] = {"algorithmic_bytes": M * k * 2 + n * k * 2 + c_bytes}
print(json.dumps({"M": M, "raster": os.environ.get("SP_GEMM_RASTER", "auto"),
                  "l2_mb": os.environ.get("SP_GEMM_L2_MB", "40"), "gemms": out}))
