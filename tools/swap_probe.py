"""Time one decode-size GEMM shape (swap-AB regime) with CUDA events.

    python tools/swap_probe.py M N K [epi] [reps]
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import ops  # noqa: E402

M, N, K = (int(x) for x in sys.argv[1:4])
epi = {"bf16": ops.EPI_STORE_BF16, "add": ops.EPI_ADD_F32, "swiglu": ops.EPI_SWIGLU, "gelu": ops.EPI_GELU,
       "f32": ops.EPI_STORE_F32, "part": ops.EPI_PARTIAL_F32}[sys.argv[4] if len(sys.argv) > 4 else "bf16"]
reps = int(sys.argv[5]) if len(sys.argv) > 5 else 20
ops.set_gemm_workspace(torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
nb = max(1, min(8, int((400 << 20) // (N * K * 2)) + 1))
bs = [torch.randn(N, K, device="cuda").to(torch.bfloat16) for _ in range(nb)]
ncol = N // 2 if epi == ops.EPI_SWIGLU else N
nslab = ops.gemm_partials(M, N, K) if epi == ops.EPI_PARTIAL_F32 else 1
d = torch.zeros(nslab * M, ncol, device="cuda",
                dtype=torch.float32 if epi in (ops.EPI_ADD_F32, ops.EPI_STORE_F32, ops.EPI_PARTIAL_F32)
                else torch.bfloat16)
for i in range(3):
    ops.gemm(a, bs[i % nb], d, epi, M=M, N=N, K=K, lda=K, ldb=K, ldd=ncol)
torch.cuda.synchronize()
# back-to-back launches captured in a CUDA graph (rotating weight copies > L2),
# so host launch overhead is excluded, as in the engine's decode graphs
n_in_graph = 16
stream = torch.cuda.Stream()
g = torch.cuda.CUDAGraph()
with torch.cuda.stream(stream):
    for i in range(2):
        ops.gemm(a, bs[i % nb], d, epi, M=M, N=N, K=K, lda=K, ldb=K, ldd=ncol)
    torch.cuda.synchronize()
    with torch.cuda.graph(g, stream=stream):
        for i in range(n_in_graph):
            ops.gemm(a, bs[i % nb], d, epi, M=M, N=N, K=K, lda=K, ldb=K, ldd=ncol)
g.replay()
torch.cuda.synchronize()
ts = []
for i in range(reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    g.replay()
    e.record()
    torch.cuda.synchronize()
    ts.append(s.elapsed_time(e) / n_in_graph)
ts.sort()
ms = ts[len(ts) // 2]
print(f"M={M} N={N} K={K} median {ms * 1e3:.1f} us/launch (graph)  weights {N * K * 2 / ms / 1e6:.0f} GB/s")
