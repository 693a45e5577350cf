"""Kernel microbenchmarks (CUDA events, warm-up, L2 flushed between reps).

    python tools/kbench.py [gemm|attn|all]
Prints one JSON line per case: shape, ms, TFLOP/s or GB/s, fraction of MEASURED_PEAKS.
"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2507_11830_b200 import ops  # noqa: E402

PEAKS = {"bf16_tflops": 1634.7, "bf16_tflops_sustained": 1366.3, "hbm_gbs": 6552.3}
try:
    PEAKS.update(json.load(open(os.path.join(os.path.dirname(__file__), "..", "MEASURED_PEAKS.json"))))
except Exception:
    pass

FLUSH = None


def flush():
    global FLUSH
    if FLUSH is None:
        FLUSH = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    FLUSH.zero_()


def timeit(fn, reps=10, warm=3, do_flush=True):
    for _ in range(warm):
        fn()
    ts = []
    for _ in range(reps):
        if do_flush:
            flush()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        fn()
        e.record()
        torch.cuda.synchronize()
        ts.append(s.elapsed_time(e))
    ts.sort()
    return ts[len(ts) // 2]


def gemm_cases():
    ops.set_gemm_workspace(torch.empty(64 << 20, dtype=torch.uint8, device="cuda"))
    M = 8192
    h, f, qkv, V = 4096, 14336, 6144, 128256
    out = []
    for name, m, n, k, epi in [("qkv", M, qkv, h, ops.EPI_STORE_BF16),
                                ("o", M, h, h, ops.EPI_ADD_F32),
                                ("gate_up", M, 2 * f, h, ops.EPI_SWIGLU),
                                ("gate_up_plain_bf16", M, 2 * f, h, ops.EPI_STORE_BF16),
                                ("n28672_k4096_f32", M, 2 * f, h, ops.EPI_STORE_F32),
                                ("down", M, h, f, ops.EPI_ADD_F32),
                                ("square8k", 8192, 8192, 8192, ops.EPI_STORE_BF16),
                                ("decode_qkv_b64", 64, qkv, h, ops.EPI_STORE_BF16),
                                ("decode_o_b64", 64, h, h, ops.EPI_ADD_F32),
                                ("decode_gate_up_b64", 64, 2 * f, h, ops.EPI_SWIGLU),
                                ("decode_down_b64", 64, h, f, ops.EPI_ADD_F32),
                                ("decode_qkv_b8", 8, qkv, h, ops.EPI_STORE_BF16),
                                ("decode_down_b8", 8, h, f, ops.EPI_ADD_F32),
                                ("decode_qkv_b256", 256, qkv, h, ops.EPI_STORE_BF16),
                                ("lm_head_b64", 64, V, h, ops.EPI_STORE_F32)]:
        a = torch.randn(m, k, device="cuda").to(torch.bfloat16)
        # rotate weight copies (> L2 in total) instead of a dirty-L2 flush
        nb = max(1, min(8, int((400 << 20) // (n * k * 2)) + 1))
        bs = [torch.randn(n, k, device="cuda").to(torch.bfloat16) for _ in range(nb)]
        b = bs[0]
        if epi == ops.EPI_SWIGLU:
            d = torch.empty(m, n // 2, device="cuda", dtype=torch.bfloat16); ldd = n // 2
        elif epi in (ops.EPI_ADD_F32, ops.EPI_STORE_F32):
            d = torch.zeros(m, n, device="cuda"); ldd = n
        else:
            d = torch.empty(m, n, device="cuda", dtype=torch.bfloat16); ldd = n
        it = [0]

        def run():
            it[0] += 1
            bb = bs[it[0] % nb]
            ops.gemm(a, bb, d, epi, M=m, N=n, K=k, lda=k, ldb=k, ldd=ldd)

        def run_ref():
            it[0] += 1
            torch.matmul(a, bs[it[0] % nb].t())
        flushing = nb == 1
        ms = timeit(run, do_flush=flushing)
        tf = 2 * m * n * k / ms / 1e9
        byts = (m * k + n * k) * 2 + d.numel() * d.element_size()
        ref_ms = timeit(run_ref, do_flush=flushing)
        del bs
        out.append(dict(kernel="gemm", case=name, M=m, N=n, K=k, ms=round(ms, 4), tflops=round(tf, 1),
                        frac_burst=round(tf / PEAKS["bf16_tflops"], 3), gbs=round(byts / ms / 1e6, 1),
                        torch_ms=round(ref_ms, 4)))
    return out


def attn_cases():
    out = []
    d, hq, hk, bs = 128, 32, 8, 64
    for T in (8192,):
        nblk = T // bs
        kpool = torch.randn(nblk, hk, bs, d, device="cuda").to(torch.bfloat16)
        vpool = torch.randn_like(kpool)
        q = torch.randn(T, hq * d, device="cuda").to(torch.bfloat16)
        bt = torch.arange(nblk, dtype=torch.int32, device="cuda").view(1, -1)
        cu = torch.tensor([0, T], dtype=torch.int32, device="cuda")
        first = torch.zeros(1, dtype=torch.int32, device="cuda")
        kvl = torch.tensor([T], dtype=torch.int32, device="cuda")
        tt = ops.attn_tile_tokens(hq, hk, d, bs)
        wl = sorted([(0, t0) for t0 in range(0, T, tt)], key=lambda w: -w[1])
        work = torch.tensor(wl, dtype=torch.int32, device="cuda").view(-1)
        o = torch.empty_like(q)
        fn = lambda: ops.attention(q, kpool, vpool, bt, cu, first, kvl, o, n_items=1, work=work,
                                   n_work=len(wl), max_q_len=T, max_kv_len=T, q_heads=hq,
                                   kv_heads=hk, head_dim=d, block_size=bs, ws=None)
        ms = timeit(fn)
        fl = 4 * d * hq * (T * (T + 1) // 2)
        out.append(dict(kernel="attn_prefill", T=T, ms=round(ms, 4), tflops=round(fl / ms / 1e9, 1)))
    for B, ctx in ((1, 2048), (64, 2048), (256, 2048)):
        nb = ctx // bs
        kpool = torch.randn(B * nb, hk, bs, d, device="cuda").to(torch.bfloat16)
        vpool = torch.randn_like(kpool)
        q = torch.randn(B, hq * d, device="cuda").to(torch.bfloat16)
        bt = torch.arange(B * nb, dtype=torch.int32, device="cuda").view(B, nb)
        cu = torch.arange(B + 1, dtype=torch.int32, device="cuda")
        kvl = torch.full((B,), ctx, dtype=torch.int32, device="cuda")
        first = kvl - 1
        ws = torch.empty(ops.attn_workspace_bytes(B, hq, d, ctx) // 4, device="cuda")
        o = torch.empty_like(q)
        fn = lambda: ops.attention(q, kpool, vpool, bt, cu, first, kvl, o, n_items=B, work=None,
                                   n_work=0, max_q_len=1, max_kv_len=ctx, q_heads=hq, kv_heads=hk,
                                   head_dim=d, block_size=bs, ws=ws)
        ms = timeit(fn)
        byts = B * ctx * hk * d * 2 * 2
        out.append(dict(kernel="attn_decode", B=B, ctx=ctx, ms=round(ms, 4), gbs=round(byts / ms / 1e6, 1),
                        frac_hbm=round(byts / ms / 1e6 / PEAKS["hbm_gbs"], 3)))
    return out


if __name__ == "__main__":
    what = sys.argv[1] if len(sys.argv) > 1 else "all"
    ops.device_check()
    res = []
    if what in ("gemm", "all"):
        res += gemm_cases()
    if what in ("attn", "all"):
        res += attn_cases()
    for r in res:
        print(json.dumps(r), flush=True)
