"""One prefill-shape GEMM launch (for ncu): python tools/gemm_one.py M N K [epi]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
ops.set_gemm_workspace(torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))  # decode split-K
epi = {"add": ops.EPI_ADD_F32, "bf16": ops.EPI_STORE_BF16,
       "f32": ops.EPI_STORE_F32}[sys.argv[4] if len(sys.argv) > 4 else "add"]
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
d = torch.zeros(M, N, device="cuda") if epi in (ops.EPI_ADD_F32, ops.EPI_STORE_F32) else \
    torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
for _ in range(3):
    ops.gemm(a, b, d, epi, M=M, N=N, K=K, lda=K, ldb=K, ldd=N)
torch.cuda.synchronize()
