"""Prefill GEMM epilogue cost: the same 8K-row projection shapes with different
epilogues (graph-replayed back to back, L2 flushed between graphs), TFLOP/s.

    python tools/epi_probe.py             # every epilogue per shape
    python tools/epi_probe.py addtma      # interleaved A/B of the TMA residual-add epilogue
    python tools/epi_probe.py storetma    # interleaved A/B of the TMA bf16-store epilogue
    python tools/epi_probe.py prod [tag]  # the four prefill projections with their production epilogues
    python tools/epi_probe.py qkvtma      # interleaved A/B of the TMA q store (QKV + RoPE epilogue)
"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import ops  # noqa: E402

ops.set_gemm_workspace(torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
M = 8192
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def bench(N, K, epi, label, reps=5, n_in=4):
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    ncol = N // 2 if epi == ops.EPI_SWIGLU else N
    dt = torch.float32 if epi in (ops.EPI_ADD_F32, ops.EPI_STORE_F32) else torch.bfloat16
    d = torch.zeros(M, ncol, device="cuda", dtype=dt)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        ops.gemm(a, b, d, epi, M=M, N=N, K=K, lda=K, ldb=K, ldd=ncol)
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n_in):
                ops.gemm(a, b, d, epi, M=M, N=N, K=K, lda=K, ldb=K, ldd=ncol)
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / n_in)
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"{label:28s} N={N:6d} K={K:6d} {ms * 1e3:8.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s", flush=True)


if len(sys.argv) > 1 and sys.argv[1] == "addtma":  # A/B of the TMA residual add, interleaved
    for rep in range(3):
        for N, K, name in ((4096, 4096, "O"), (4096, 14336, "down")):
            for on in ("0", "1"):
                os.environ["SP_ADD_TMA"] = on
                bench(N, K, ops.EPI_ADD_F32, f"{name} add_f32 add_tma={on}")
    sys.exit(0)
def bench_qkv_rope(label, reps=5, n_in=4, hq=32, hk=8, K=4096, bs=64):
    from paper_2507_11830_b200.weights import rope_table
    N = (hq + 2 * hk) * 128
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = (torch.randn(N, K, device="cuda") * 0.02).to(torch.bfloat16)
    pos = torch.arange(M, dtype=torch.int32, device="cuda")
    slot = torch.arange(M, dtype=torch.int32, device="cuda")
    tab = torch.from_numpy(rope_table(M, 128, 500000.0, None)).cuda()
    q = torch.empty(M, hq * 128, device="cuda", dtype=torch.bfloat16)
    kp = torch.empty(M // bs, hk, bs, 128, device="cuda", dtype=torch.bfloat16)
    vp = torch.empty_like(kp)

    def run():
        ops.gemm_qkv_rope(a, b, M=M, K=K, lda=K, ldb=K, pos=pos, slot=slot, rope=tab, q_out=q,
                          k_pool=kp, v_pool=vp, q_heads=hq, kv_heads=hk, block_size=bs)
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        run()
        torch.cuda.synchronize()
        with torch.cuda.graph(g, stream=s):
            for _ in range(n_in):
                run()
    ts = []
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.replay()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / n_in)
    ts.sort()
    ms = ts[len(ts) // 2]
    print(f"{label:28s} N={N:6d} K={K:6d} {ms * 1e3:8.1f} us  {2 * M * N * K / ms / 1e9:7.1f} TFLOP/s", flush=True)


if len(sys.argv) > 1 and sys.argv[1] == "prod":  # the four prefill projections as the engine runs them
    tag = sys.argv[2] if len(sys.argv) > 2 else ""
    bench_qkv_rope(f"{tag} QKV rope")
    bench(4096, 4096, ops.EPI_ADD_F32, f"{tag} O add_f32")
    bench(28672, 4096, ops.EPI_SWIGLU, f"{tag} gate_up swiglu")
    bench(4096, 14336, ops.EPI_ADD_F32, f"{tag} down add_f32")
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "qkvtma":  # A/B of the TMA q store in the QKV+RoPE epilogue
    for rep in range(3):
        for on in ("0", "1"):
            os.environ["SP_STORE_TMA"] = on
            bench_qkv_rope(f"QKV rope store_tma={on}")
    sys.exit(0)
if len(sys.argv) > 1 and sys.argv[1] == "storetma":  # A/B of the TMA bf16 store, interleaved
    for rep in range(3):
        for N, K, name, epi in ((28672, 4096, "gate_up swiglu", ops.EPI_SWIGLU),
                                (6144, 4096, "QKV bf16", ops.EPI_STORE_BF16)):
            for on in ("0", "1"):
                os.environ["SP_STORE_TMA"] = on
                bench(N, K, epi, f"{name} store_tma={on}")
    sys.exit(0)
for N, K, name in ((4096, 4096, "O"), (4096, 14336, "down"), (6144, 4096, "QKV"), (28672, 4096, "gate_up")):
    for epi, en in ((ops.EPI_STORE_BF16, "bf16"), (ops.EPI_STORE_F32, "f32"), (ops.EPI_ADD_F32, "add_f32"),
                    (ops.EPI_SWIGLU, "swiglu")):
        bench(N, K, epi, f"{name} {en}")
